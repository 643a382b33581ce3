#!/usr/bin/env bash
# qkv split count under the long-K down rule (4-layer L3 decode forward)
export PYTHONPATH=$PWD
out=gpurun_out/split_sweep2.log
for T in 64 32 16; do
  for cfg in "" "6144:4096:3" "6144:4096:2" "6144:4096:8"; do
    for rep in 1 2; do
      echo -n "T=$T PL_SPLITS=$cfg rep=$rep : " >> $out
      PL_SPLITS=$cfg timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
    done
  done
done
