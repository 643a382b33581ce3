#!/usr/bin/env bash
# 4-layer L3 decode forward at T = 16/32/64 (A/B for reduce-kernel changes)
export PYTHONPATH=$PWD
out=${1:-gpurun_out/reduce_ab.log}
for T in 16 32 64; do
  for rep in 1 2 3; do
    echo -n "T=$T rep=$rep : " >> $out
    timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
  done
done
