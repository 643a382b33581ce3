#!/bin/bash
# tcgen05 prefill attention: XU-pipe offload variants (ex2 on FMA, bf16 convert on ALU), A/B
cd "$(dirname "$0")/.."
O=gpurun_out/attn_q1
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
P=paper_2507_05043_b200
for v in "q1:-DPL_AT_QBUF=1" "q1k3:-DPL_AT_QBUF=1 -DPL_AT_KST=3" "q1v3:-DPL_AT_QBUF=1 -DPL_AT_VST=3"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p $P/_build_$name
  for f in $P/_build/*.o; do [ "$(basename $f)" != attn_tc.o ] && cp -p $f $P/_build_$name/; done
  PL_BUILD_VARIANT=$name PL_NVCC_EXTRA="$flags" python -m paper_2507_05043_b200.build >> $O/build.log 2>&1
done
timeout 300 python scripts/bench_attn.py > $O/bench_base.log 2>&1
for name in q1 q1k3 q1v3; do
  PL_LIB_PATH=$P/_lib_$name/libb200link.so timeout 120 python scripts/attn_debug.py 2 32 8 512,1000,37,2048 >> $O/cases.log 2>&1
  PL_LIB_PATH=$P/_lib_$name/libb200link.so timeout 300 python scripts/bench_attn.py > $O/bench_$name.log 2>&1
done
echo done > $O/done
