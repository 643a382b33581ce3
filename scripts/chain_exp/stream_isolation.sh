#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
B220="-DCH_BUDGET_KB=220 -DCH_BS16=8 -DCH_BS32=8 -DCH_BS64=6 -DCH_BS128=4 -DCH_BS256=2"
declare -A V
V[nomma]="-DCH_EXP_NOMMA"
V[nomma220]="-DCH_EXP_NOMMA $B220"
V[nob]="-DCH_EXP_NOB"
V[nob220]="-DCH_EXP_NOB $B220"
V[nomma_nob220]="-DCH_EXP_NOMMA -DCH_EXP_NOB $B220"
V[b220]="$B220"
for v in "${!V[@]}"; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m paper_2507_05043_b200.build > gpurun_out/build_$v.log 2>&1 &
done
wait
for v in base b220 nomma nomma220 nob nob220 nomma_nob220; do
  lib=""
  [ "$v" != base ] && lib="$PWD/paper_2507_05043_b200/_lib_$v/libb200link.so"
  PL_LIB_PATH=$lib timeout 300 python scripts/chain_bench.py --tag $v >> gpurun_out/chain_bench2.log 2>&1
done
