#!/bin/bash
# 4-GPU box, one process: copied vs fused decode hops with link recording off in both
# arms, a link-recorded run for the chunk log, the live NVLink demo, the CLI backend
cd "$(dirname "$0")/.."
O=gpurun_out/stages3
mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
T="timeout 900"
$T python scripts/run_stages.py --stages 8 --gpus 4 --no-links > $O/s8_g4_copy.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 4 --fuse --no-links > $O/s8_g4_fused.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 --no-links > $O/s4_g4_copy.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 --fuse --no-links > $O/s4_g4_fused.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 > $O/s4_g4_links.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
  --master-port 29631 scripts/check_live.py > $O/check_live2.log 2>&1
$T python -m pytest tests/test_multigpu_gpu.py tests/test_cli_backend.py -q -m gpu > $O/pytest.log 2>&1
echo done > $O/done
