#!/bin/bash
# cluster split-K for the residual GEMMs too (PL_CSK=7: o / down reduce their split-K tile
# over DSMEM with the vectorised epilogue, then the norm-only kernel) vs the default
# (PL_CSK=5: partials + the residual+norm reduce kernel): parity, 4-layer forward, bench
cd "$(dirname "$0")/.."
O=gpurun_out/csk7; rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m $P.build > $O/build.log 2>&1
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build > $O/build_tl.log 2>&1 &
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullmodel_parity_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
PL_CSK=7 timeout 900 python -m pytest tests/test_fullmodel_parity_gpu.py tests/test_pipeline_gpu.py -m gpu -q -x > $O/pytest_csk7.log 2>&1
wait
for rep in 1 2 3; do
for T in 64 32; do
  for m in 5 7; do
    echo -n "csk=$m T=$T rep=$rep: " >> $O/layers.log
    PL_CSK=$m timeout 300 python scripts/profile_decode.py --layers 4 --T $T --ctx 640 --iters 20 --last 0 2>&1 | tail -1 >> $O/layers.log
  done
done
done
PL_CSK=7 PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T 64 --ctx 640 > $O/tl_T64_csk7.log 2>&1
for m in 5 7; do
  echo "== csk=$m" >> $O/bench.log
  PL_CSK=$m timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | tail -1 | cut -c1-330 >> $O/bench.log
done
echo done > $O/done
