#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
python scripts/profile_decode.py --layers 2 --T 64 --iters 2 --last 0 > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 2 \
    -o gpurun_out/chain_prof python scripts/profile_decode.py --layers 2 --T 64 --iters 2 --last 0 > gpurun_out/ncu_full.log 2>&1
