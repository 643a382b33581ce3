#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
declare -A V
V[ctas2]="-DCH_CTAS=2 -DCH_BS16=6 -DCH_BS32=4 -DCH_BS64=3 -DCH_BS128=2 -DCH_BS256=2"
V[ctas2b]="-DCH_CTAS=2 -DCH_BUDGET_KB=108 -DCH_BS16=4 -DCH_BS32=4 -DCH_BS64=2 -DCH_BS128=2 -DCH_BS256=2"
for v in "${!V[@]}"; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m paper_2507_05043_b200.build > gpurun_out/build_$v.log 2>&1 &
done
wait
for v in base ctas2 ctas2b; do
  lib=""
  [ "$v" != base ] && lib="$PWD/paper_2507_05043_b200/_lib_$v/libb200link.so"
  PL_LIB_PATH=$lib timeout 300 python scripts/chain_bench.py --tag $v >> gpurun_out/chain_bench3.log 2>&1
  for T in 64 16 8; do
    echo "$v T=$T: $(PL_LIB_PATH=$lib timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/ring3.log
  done
done
