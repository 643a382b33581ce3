#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
for k in 7 8; do
  PL_CHAIN_TRACE=$k timeout 300 python scripts/chain_trace.py gpurun_out/trace_$k.npz > gpurun_out/trace_$k.log 2>&1
done
PL_CHAIN_TRACE=8 timeout 300 python scripts/chain_trace.py gpurun_out/trace_8_T8.npz --T 8 > gpurun_out/trace_8_T8.log 2>&1
for T in 64 8; do
  echo "T=$T chain=1: $(PL_CHAIN=1 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
done
