#!/bin/bash
# timeline of a 4-layer L3 decode forward at T = 64 (cluster split-K phases)
cd "$(dirname "$0")/.."
O=gpurun_out/tl64; rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build > $O/build.log 2>&1
PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T 64 --ctx 640 > $O/tl_T64.log 2>&1
PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T 32 --ctx 640 > $O/tl_T32.log 2>&1
echo done > $O/done
