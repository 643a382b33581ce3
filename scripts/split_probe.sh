#!/usr/bin/env bash
# ncu durations of the split-K GEMM and its reduce for several split counts
export PYTHONPATH=$PWD
for shape in 4096,14336 4096,4096 6144,4096; do
  for s in 3 4 5 6 8 9; do
    PL_SPLITK_FORCE=$s ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 8 --csv \
      --log-file gpurun_out/split_${shape/,/x}_s$s.csv python scripts/bench_gemm.py --T 64 --shapes $shape \
      > /dev/null 2>&1
  done
done
