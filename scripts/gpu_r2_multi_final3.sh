#!/bin/bash
# end-of-round multi-GPU evidence on a 4-GPU box (final code): NCCL checks, N = 2 / 4
# bench lines, 8 / 4 stages in one process, multi-GPU + CLI tests
cd "$(dirname "$0")/.."
O=gpurun_out/multi_final3
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
T="timeout 900"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T $TR --nproc-per-node 2 --master-port 29521 scripts/check_multigpu.py --model tiny > $O/check_n2.log 2>&1
$T $TR --nproc-per-node 4 --master-port 29522 scripts/check_multigpu.py --model l3-2 --stages 4 --requests 8 --prompt 96 --decode 8 > $O/check_n4.log 2>&1
$T $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2.log 2>&1
$T $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 3 --warmup 3 > $O/bench_n4.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 4 --no-links > $O/s8_g4.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 4 --no-links > $O/s8_g4_rep2.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 > $O/s4_g4_links.log 2>&1
$T python -m pytest tests/test_multigpu_gpu.py tests/test_cli_backend.py -q -m gpu > $O/pytest.log 2>&1
echo done > $O/done
