#!/bin/bash
# final-code evidence: ncu --set full of the decode o / qkv GEMMs and the decode attention
# (4-layer L3 decode forward, T = 64), and two more N=1 bench runs for the box spread
cd "$(dirname "$0")/.."
O=gpurun_out/evidence; rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
CMD="python scripts/profile_decode.py --layers 4 --iters 2 --last 0"
$CMD > $O/plain.log 2>&1 || { echo fail > $O/done; exit 0; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 9 -c 1 -o $O/o_proj_T64 $CMD > $O/ncu_o.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 8 -c 1 -o $O/qkv_T64 $CMD > $O/ncu_qkv.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 2 -c 1 -o $O/attn_T64 $CMD > $O/ncu_attn.log 2>&1
for r in 1 2; do
  timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n1_rep$r.log 2>&1
done
echo done > $O/done
