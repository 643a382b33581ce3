#!/bin/bash
# one ncu --set full capture of the tcgen05 prefill attention kernel (4 x 2048, L3 heads)
cd "$(dirname "$0")/.."
O=gpurun_out/attn_ncu
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc_kernel -c 1 \
  -o $O/attn_tc python scripts/attn_debug.py 2 32 8 $(python -c "print(','.join(['512']*64))") > $O/ncu.log 2>&1
echo done > $O/done
