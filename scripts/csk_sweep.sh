#!/usr/bin/env bash
# decode forward (4 L3 layers) under cluster split-K masks (PL_CSK: 1 qkv, 2 residual+norm, 4 plain)
export PYTHONPATH=$PWD
for T in 16 64; do
  for C in 0 1 2 3 7; do
    echo -n "PL_CSK=$C T=$T : " >> gpurun_out/csk.log
    PL_CSK=$C timeout 120 python scripts/profile_decode.py --layers 4 --iters 4 --last 0 --T $T 2>&1 | tail -1 >> gpurun_out/csk.log
  done
done
