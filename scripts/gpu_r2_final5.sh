#!/bin/bash
# round-2 final validation (final code incl. epilogue helper warps) on one B200: GPU suite, smoke,
# N=1 bench, reference arm, decode launch list, ncu --set full of the decode gate_up GEMM,
# per-CTA kernel timeline at T = 64 / 16 / 1
cd "$(dirname "$0")/.."
O=gpurun_out/final5
rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m $P.build > $O/build.log 2>&1
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build >> $O/build.log 2>&1 &
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_n1.log 2>&1
echo "bench rc=$?" >> $O/bench_n1.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1
wait
for T in 64 16 1; do
  PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T $T --ctx 640 > $O/tl_T$T.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --decode 8 --no-cpu-baseline --no-parity"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"gemm_tc_kernel|attn_decode|reduce_|rmsnorm|embed|argmax|token_scatter" -s 3000 -c 1200 --csv \
    --log-file $O/launches_decode.csv $CMD > $O/launches_decode_run.log 2>&1
timeout 300 python scripts/profile_decode.py --layers 4 --iters 2 --last 0 > $O/decode_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 10 -c 1 \
    -o $O/gate_up_T64 python scripts/profile_decode.py --layers 4 --iters 2 --last 0 > $O/ncu_gate_up.log 2>&1
echo done > $O/done
