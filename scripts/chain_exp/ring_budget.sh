#!/bin/bash
# chain kernel ring experiments: bigger shared-memory budget, ring splits
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
declare -A V
V[b220a]="-DCH_BUDGET_KB=220 -DCH_BS16=8 -DCH_BS32=8 -DCH_BS64=6 -DCH_BS128=4 -DCH_BS256=2"
V[b220b]="-DCH_BUDGET_KB=220 -DCH_BS16=12 -DCH_BS32=10 -DCH_BS64=4 -DCH_BS128=3 -DCH_BS256=2"
V[b220c]="-DCH_BUDGET_KB=220 -DCH_BS16=16 -DCH_BS32=12 -DCH_BS64=8 -DCH_BS128=5 -DCH_BS256=3"
for v in b220a b220b b220c; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m paper_2507_05043_b200.build > gpurun_out/build_$v.log 2>&1 &
done
wait
for v in base b220a b220b b220c; do
  lib=""
  [ "$v" != base ] && lib="$PWD/paper_2507_05043_b200/_lib_$v/libb200link.so"
  for T in 64 16 8; do
    echo "$v T=$T: $(PL_LIB_PATH=$lib timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/ring2.log
  done
done
