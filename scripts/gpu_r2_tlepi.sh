#!/bin/bash
# timeline with epilogue-end stamps (GEMM p4 = warp 2's epilogue done, p5 = thread 0 at the final barrier)
cd "$(dirname "$0")/.."
O=gpurun_out/tlepi; rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build > $O/build.log 2>&1
for T in 64 32; do
  PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T $T --ctx 640 > $O/tl_T$T.log 2>&1
done
echo done > $O/done
