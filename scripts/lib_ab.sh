#!/usr/bin/env bash
# Same-box A/B of two builds of libb200link.so (ab/old.so vs ab/new.so, git-ignored):
# 4-layer L3 decode forward at T = 16/32/64, alternating builds
export PYTHONPATH=$PWD
out=${1:-gpurun_out/lib_ab.log}
lib=paper_2507_05043_b200/_lib/libb200link.so
cp $lib /tmp/keep.so
for rep in 1 2 3; do
  for v in old new; do
    cp ab/$v.so $lib
    for T in 16 32 64; do
      echo -n "$v T=$T rep=$rep : " >> $out
      timeout 120 python scripts/profile_decode.py --layers 4 --iters 6 --last 0 --T $T 2>&1 | tail -1 >> $out
    done
  done
done
cp /tmp/keep.so $lib
