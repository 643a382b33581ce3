#!/bin/bash
# round 2 multi-GPU evidence on a 4-GPU box: single-process 8 stages on 4 / 1 GPUs,
# NCCL checks with realized chunk logs, bench at N = 2 / 4, NCCL channel bound
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/multi
python -m paper_2507_05043_b200.build > gpurun_out/multi/build.log 2>&1
nvidia-smi topo -m > gpurun_out/multi/topo.txt 2>&1
T="timeout 900"
$T python scripts/run_stages.py --stages 8 --gpus 4 > gpurun_out/multi/stages8_gpus4.log 2>&1
$T python scripts/run_stages.py --stages 8 --gpus 1 > gpurun_out/multi/stages8_gpus1.log 2>&1
$T python scripts/run_stages.py --stages 4 --gpus 4 > gpurun_out/multi/stages4_gpus4.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO $T $TR --nproc-per-node 2 --master-port 29511 scripts/check_multigpu.py --model tiny > gpurun_out/multi/check_n2.log 2>&1
$T $TR --nproc-per-node 4 --master-port 29512 scripts/check_multigpu.py --model l3-2 --stages 4 --requests 8 --prompt 96 --decode 8 > gpurun_out/multi/check_n4.log 2>&1
$T $TR --nproc-per-node 2 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/multi/bench_n2.log 2>&1
$T $TR --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/multi/bench_n4.log 2>&1
NCCL_MAX_NCHANNELS=2 $T $TR --nproc-per-node 4 --master-port 29515 bench.py --gpus 4 --steps 3 --warmup 3 --no-parity --no-cpu-baseline > gpurun_out/multi/bench_n4_nch2.log 2>&1
$T python -m pytest tests/test_multigpu_gpu.py -q -m gpu > gpurun_out/multi/pytest_multigpu.log 2>&1
echo done > gpurun_out/multi/done
