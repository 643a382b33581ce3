#!/usr/bin/env bash
# decode forward time vs micro-batch size and fusion (4 L3 layers, ctx 640)
export PYTHONPATH=$PWD
for T in 1 8 16 32 64 128; do
  echo -n "T=$T fuse=1: " >> gpurun_out/layer.log; python scripts/profile_decode.py --layers 4 --iters 4 --last 0 --T $T 2>&1 | tail -1 >> gpurun_out/layer.log
done
echo -n "T=64 fuse=0: " >> gpurun_out/layer.log; PL_FUSE=0 python scripts/profile_decode.py --layers 4 --iters 4 --last 0 --T 64 2>&1 | tail -1 >> gpurun_out/layer.log
echo -n "T=64 ctx=64: " >> gpurun_out/layer.log; python scripts/profile_decode.py --layers 4 --iters 4 --last 0 --T 64 --ctx 64 2>&1 | tail -1 >> gpurun_out/layer.log
