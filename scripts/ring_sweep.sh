#!/usr/bin/env bash
export PYTHONPATH=$PWD
run() { echo -n "$* : " >> gpurun_out/ring.log; env "$@" python scripts/profile_decode.py --layers 4 --iters 4 --last 0 2>&1 | tail -1 >> gpurun_out/ring.log; }
run PL_X=0
run PL_GEMM_WIDE=1
run PL_GEMM_WIDE=1 PL_SPLIT_RULE=fit
run PL_SPLIT_RULE=fit
for w in 0 1; do echo "wide=$w" >> gpurun_out/ring_bg.log; PL_GEMM_WIDE=$w python scripts/bench_gemm.py --T 16 64 >> gpurun_out/ring_bg.log 2>&1; done
