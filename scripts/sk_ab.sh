#!/usr/bin/env bash
# 4-layer L3 decode forward at T = 16/32/64: default split-K vs DP + stream-K hybrid vs stream-K
export PYTHONPATH=$PWD
out=${1:-gpurun_out/sk_ab.log}
for rep in 1 2; do
  for m in "PL_X=0" "PL_SK_HYBRID=1" "PL_STREAMK=1"; do
    for T in 16 32 64; do
      echo -n "$m T=$T rep=$rep : " >> $out
      env $m timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
    done
  done
done
