#!/bin/bash
# decode epilogues (SwiGLU lane split, batched qkv RoPE/KV-append loads): kernel parity,
# 4-layer decode forward, timeline, N=1 bench
cd "$(dirname "$0")/.."
O=gpurun_out/epi
rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m $P.build > $O/build.log 2>&1
PL_BUILD_VARIANT=tl PL_NVCC_EXTRA="-DPL_TIMELINE" python -m $P.build >> $O/build.log 2>&1 &
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullmodel_parity_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
wait
for rep in 1 2; do
for T in 64 32 16 1; do
  echo -n "rep=$rep T=$T: " >> $O/layers.log
  timeout 300 python scripts/profile_decode.py --layers 4 --T $T --ctx 640 --iters 20 --last 0 2>&1 | tail -1 >> $O/layers.log
done
done
for T in 64 32 1; do
  PL_LIB_PATH=$PWD/$P/_lib_tl/libb200link.so timeout 300 python scripts/timeline.py --layers 4 --T $T --ctx 640 > $O/tl_T$T.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 > $O/bench.log 2>&1
echo done > $O/done
