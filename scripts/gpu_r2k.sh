#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
declare -A V
V[nomma]="-DCH_EXP_NOMMA"
V[b220]="-DCH_BUDGET_KB=220 -DCH_BS16=8 -DCH_BS32=8 -DCH_BS64=6 -DCH_BS128=4 -DCH_BS256=2"
for v in nomma b220; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m paper_2507_05043_b200.build > gpurun_out/build_$v.log 2>&1 &
done
wait
for v in base nomma b220; do
  lib=""
  [ "$v" != base ] && lib="$PWD/paper_2507_05043_b200/_lib_$v/libb200link.so"
  PL_LIB_PATH=$lib timeout 300 python scripts/chain_bench.py --tag $v >> gpurun_out/chain_bench.log 2>&1
done
