#!/usr/bin/env bash
# decode forward (4 L3 layers, T=64) under GEMM grid / split policies
export PYTHONPATH=$PWD
run() { echo -n "$* : " >> gpurun_out/grid.log; env "$@" python scripts/profile_decode.py --layers 4 --iters 4 --last 0 2>&1 | tail -1 >> gpurun_out/grid.log; }
run PL_X=0
run PL_SPLIT_RULE=fit PL_GRID_PER_SM=1
run PL_SPLIT_RULE=fit
run PL_GRID_PER_SM=1
run PL_GEMM_WIDE=1
run PL_SPLIT_RULE=fit PL_GEMM_WIDE=1
run PL_STREAMK=1
run PL_PDL=0
