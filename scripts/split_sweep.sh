#!/usr/bin/env bash
# 4-layer L3 decode forward under per-shape split-K overrides (PL_SPLITS="N:K:s,...")
# qkv = 6144:4096, o = 4096:4096, down = 4096:14336 (defaults 4 / 5 / 5)
export PYTHONPATH=$PWD
out=gpurun_out/split_sweep.log
for T in 16 64 32; do
  for cfg in "" "4096:4096:8" "4096:14336:8" "4096:4096:8,4096:14336:8" "6144:4096:6" \
             "6144:4096:6,4096:4096:8,4096:14336:8" "4096:14336:9" "4096:4096:4,4096:14336:4"; do
    for rep in 1 2; do
      echo -n "T=$T PL_SPLITS=$cfg rep=$rep : " >> $out
      PL_SPLITS=$cfg timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
    done
  done
done
