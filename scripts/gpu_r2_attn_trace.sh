#!/bin/bash
# timeline of one CTA of the tcgen05 prefill attention (experiment build -DPL_AT_TRACE)
cd "$(dirname "$0")/.."
O=gpurun_out/attn_trace
rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
mkdir -p $P/_build_trace
for f in $P/_build/*.o; do [ "$(basename $f)" != attn_tc.o ] && cp -p $f $P/_build_trace/; done
PL_BUILD_VARIANT=trace PL_NVCC_EXTRA="-DPL_AT_TRACE" python -m paper_2507_05043_b200.build >> $O/build.log 2>&1
L=$PWD/$P/_lib_trace/libb200link.so
PL_LIB_PATH=$L timeout 120 python scripts/attn_trace.py 32 8 8192 > $O/trace_1x8192.log 2>&1
PL_LIB_PATH=$L timeout 120 python scripts/attn_trace.py 32 8 $(python -c "print(','.join(['512']*64))") > $O/trace_64x512.log 2>&1
echo done > $O/done
