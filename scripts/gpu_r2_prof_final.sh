#!/bin/bash
# final ncu evidence: decode-phase launch list of a serving run (GEMM / attention / reduce
# kernels only) and one --set full capture of the tcgen05 prefill attention kernel
cd "$(dirname "$0")/.."
O=gpurun_out/prof_final
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --decode 8 --no-cpu-baseline --no-parity"
timeout 600 $CMD > $O/plain.log 2>&1 || { echo "plain run failed" > $O/done; exit 0; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"gemm_tc_kernel|attn_decode|reduce_|rmsnorm|embed|argmax|token_scatter" -s 3000 -c 1200 --csv \
    --log-file $O/launches_decode.csv $CMD > $O/launches_decode_run.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc_kernel -c 1 \
    -o $O/attn_tc_4x2048 python scripts/attn_debug.py 2 32 8 2048,2048,2048,2048 > $O/ncu_attn.log 2>&1
echo done > $O/done
