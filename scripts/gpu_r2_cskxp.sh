#!/bin/bash
# which part of the cluster split-K RoPE epilogue is slow: timing-only variants that drop
# the metadata / RoPE-table loads (nometa) or the DSMEM partial loads (nodsmem)
cd "$(dirname "$0")/.."
O=gpurun_out/cskxp; rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
declare -A V
V[tl]="-DPL_TIMELINE"
V[tlnometa]="-DPL_TIMELINE -DPL_XP_NOMETA"
V[tlnodsmem]="-DPL_TIMELINE -DPL_XP_NODSMEM"
for v in tl tlnometa tlnodsmem; do
  PL_BUILD_VARIANT=$v PL_NVCC_EXTRA="${V[$v]}" python -m $P.build > $O/build_$v.log 2>&1 &
done
wait
for v in tl tlnometa tlnodsmem; do
  PL_LIB_PATH=$PWD/$P/_lib_$v/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T 64 --ctx 640 > $O/$v.log 2>&1
done
echo done > $O/done
