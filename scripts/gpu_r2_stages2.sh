#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/stages2
python -m paper_2507_05043_b200.build > gpurun_out/stages2/build.log 2>&1
T="timeout 900"
$T python scripts/run_stages.py --fuse --stages 8 --gpus 4 > gpurun_out/stages2/s8_g4.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 4 --no-links > gpurun_out/stages2/s8_g4_nofuse.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 > gpurun_out/stages2/s4_g4.log 2>&1
$T python -m pytest tests/test_multigpu_gpu.py tests/test_cli_backend.py -q -m gpu > gpurun_out/stages2/pytest.log 2>&1
echo done > gpurun_out/stages2/done
