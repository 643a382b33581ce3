#!/usr/bin/env bash
# decode forward time (4 L3 layers, T=64, PDL chain) vs cross-kernel L2 weight prefetch depth
export PYTHONPATH=$PWD
for mb in 64 256; do
  for pf in 0 16 64 256 4096; do
    echo -n "maxmb=$mb pf=$pf " >> gpurun_out/l2pf.log
    PL_L2PF=$pf PL_L2PF_MAXMB=$mb python scripts/profile_decode.py --layers 4 --iters 4 --last 0 2>&1 | tail -1 >> gpurun_out/l2pf.log
  done
done
