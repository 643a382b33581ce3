#!/bin/bash
# per-CTA %globaltimer timeline of a 4-layer L3 decode forward (PDL chain) at T = 64 / 16 / 1
cd "$(dirname "$0")/.."
O=gpurun_out/timeline
rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m $P.build > $O/build.log 2>&1
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build >> $O/build.log 2>&1
for T in 64 16 1; do
  PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T $T --ctx 640 > $O/T$T.log 2>&1
done
echo done > $O/done
