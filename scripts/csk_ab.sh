#!/usr/bin/env bash
# 4-layer L3 decode forward at T = 32/64 under cluster split-K masks (PL_CSK)
export PYTHONPATH=$PWD
out=${1:-gpurun_out/csk_ab.log}
for T in 32 64; do
  for m in 5 4 7; do
    for rep in 1 2; do
      echo -n "T=$T PL_CSK=$m rep=$rep : " >> $out
      PL_CSK=$m timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
    done
  done
done
