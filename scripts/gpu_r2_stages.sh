#!/bin/bash
# 8 stages in one process on 4 GPUs / 1 GPU (two stages per GPU), fused vs copied decode hops
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/stages
python -m paper_2507_05043_b200.build > gpurun_out/stages/build.log 2>&1
T="timeout 900"
$T python scripts/run_stages.py --fuse --stages 8 --gpus 4 > gpurun_out/stages/s8_g4.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 4 --no-links > gpurun_out/stages/s8_g4_nofuse.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 > gpurun_out/stages/s4_g4.log 2>&1
$T python scripts/run_stages.py --fuse --stages 8 --gpus 1 > gpurun_out/stages/s8_g1.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 1 --no-links > gpurun_out/stages/s8_g1_nofuse.log 2>&1
$T python -m pytest tests/test_pipeline_gpu.py -q -m gpu -k "fused_transport or realized or throttle" > gpurun_out/stages/pytest.log 2>&1
echo done > gpurun_out/stages/done
