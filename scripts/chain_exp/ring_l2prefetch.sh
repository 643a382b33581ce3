#!/bin/bash
# chain kernel ring experiments: variant builds, 4-layer decode forward at T = 64 / 8
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
declare -A V
V[base]=""
V[pf8]="-DCH_L2PF=8"
V[pf16]="-DCH_L2PF=16"
V[bs4]="-DCH_BS16=8 -DCH_BS32=6 -DCH_BS64=4 -DCH_BS128=3 -DCH_BS256=2"
V[bs4pf8]="-DCH_BS16=8 -DCH_BS32=6 -DCH_BS64=4 -DCH_BS128=3 -DCH_BS256=2 -DCH_L2PF=8"
for v in pf8 pf16 bs4 bs4pf8; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m paper_2507_05043_b200.build > gpurun_out/build_$v.log 2>&1 &
done
wait
for v in base pf8 pf16 bs4 bs4pf8; do
  lib=""
  [ "$v" != base ] && lib="$PWD/paper_2507_05043_b200/_lib_$v/libb200link.so"
  for T in 64 8; do
    echo "$v T=$T: $(PL_LIB_PATH=$lib timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/ring.log
  done
done
PL_CHAIN=1 python scripts/profile_decode.py --layers 4 --T 64 --iters 2 --last 0 > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_chain2.csv \
  python scripts/profile_decode.py --layers 4 --T 64 --iters 2 --last 0 > gpurun_out/ncu_chain2.log 2>&1
