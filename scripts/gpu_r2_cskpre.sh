#!/bin/bash
# cluster split-K QKV epilogue: base = 16-byte DSMEM loads (4 features per thread) with the
# RoPE/KV metadata preloaded by the idle epilogue warps during the main loop; nov4 = one
# feature per thread (scalar DSMEM loads), preloaded; old = scalar, loaded after the main loop
# (PL_CSK_V4=0 PL_CSK_PRELOAD=0): parity, 4-layer forward, bench
cd "$(dirname "$0")/.."
O=gpurun_out/cskpre; rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m $P.build > $O/build.log 2>&1
PL_BUILD_VARIANT=nov4 PL_NVCC_EXTRA="-DPL_CSK_V4=0" python -m $P.build > $O/build_nov4.log 2>&1 &
PL_BUILD_VARIANT=old PL_NVCC_EXTRA="-DPL_CSK_V4=0 -DPL_CSK_PRELOAD=0" python -m $P.build > $O/build_old.log 2>&1 &
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build > $O/build_tl.log 2>&1 &
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullmodel_parity_gpu.py tests/test_pipeline_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
wait
for rep in 1 2 3; do
for T in 64 32; do
  for v in base nov4 old; do
    lib=""; [ "$v" != base ] && lib="$PWD/$P/_lib_$v/libb200link.so"
    echo -n "$v T=$T rep=$rep: " >> $O/layers.log
    PL_LIB_PATH=$lib timeout 300 python scripts/profile_decode.py --layers 4 --T $T --ctx 640 --iters 20 --last 0 2>&1 | tail -1 >> $O/layers.log
  done
done
done
PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T 64 --ctx 640 > $O/tl_T64.log 2>&1
for v in base old; do
  lib=""; [ "$v" != base ] && lib="$PWD/$P/_lib_$v/libb200link.so"
  echo "== $v" >> $O/bench.log
  PL_LIB_PATH=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | tail -1 | cut -c1-330 >> $O/bench.log
done
echo done > $O/done
