#!/usr/bin/env bash
# ncu evidence for profiles/ (run on a GPU box from the repo root, one GPU):
#   1. the bench command once without ncu (must exit 0)
#   2. its launch list inside the timed region (gpu__time_duration, cold-cache, serialised)
#   3. --set full captures of the top decode kernels (gate_up GEMM, attention, o GEMM)
# Outputs land in gpurun_out/prof_<tag>*; summarise here with scripts/summarize_ncu.py.
set -u
TAG=${1:-r1}
OUT=gpurun_out
export PYTHONPATH=$PWD
# launch list of a short serving run (decode 4 tokens) -- the full 256-token bench
# command is ~270k launches and does not finish under ncu; the decode kernel set and
# per-step structure are the same.  Skip setup, profiling and the warm-up runs.
CMD="python bench.py --steps 1 --warmup 3 --decode 4 --no-cpu-baseline"
$CMD > $OUT/prof_${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 14000 -c 1500 --csv \
    --log-file $OUT/prof_${TAG}_launches.csv $CMD > $OUT/prof_${TAG}_launches_run.log 2>&1
python scripts/profile_decode.py --layers 4 --iters 2 --last 0 > $OUT/prof_${TAG}_decode_plain.log 2>&1 || exit 1
# per 4-layer decode forward: gemm launches qkv,o,gate_up,down per layer; skip the first forwards
ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 10 -c 1 \
    -o $OUT/prof_${TAG}_gate_up python scripts/profile_decode.py --layers 4 --iters 2 --last 0 \
    > $OUT/prof_${TAG}_gate_up.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 9 -c 1 \
    -o $OUT/prof_${TAG}_o_proj python scripts/profile_decode.py --layers 4 --iters 2 --last 0 \
    > $OUT/prof_${TAG}_o_proj.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 2 -c 1 \
    -o $OUT/prof_${TAG}_attn python scripts/profile_decode.py --layers 4 --iters 2 --last 0 \
    > $OUT/prof_${TAG}_attn.log 2>&1
echo done
