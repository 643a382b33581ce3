#!/bin/bash
# decode attention: balanced persistent grid vs min(items, 2 x SMs), 4-layer L3 decode forward
cd "$(dirname "$0")/.."
O=gpurun_out/attn_dec
rm -rf $O; mkdir -p $O
P=paper_2507_05043_b200
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
mkdir -p $P/_build_nobal
for f in $P/_build/*.o; do [ "$(basename $f)" != attention.o ] && cp -p $f $P/_build_nobal/; done
PL_BUILD_VARIANT=nobal PL_NVCC_EXTRA="-DPL_ATTN_BALANCE=0" python -m paper_2507_05043_b200.build >> $O/build.log 2>&1
for rep in 1 2; do
for T in 64 32 8; do
  for v in base nobal; do
    lib=""; [ "$v" != base ] && lib="$PWD/$P/_lib_$v/libb200link.so"
    echo -n "$v T=$T rep=$rep: " >> $O/layers.log
    PL_LIB_PATH=$lib timeout 300 python scripts/profile_decode.py --layers 4 --T $T --ctx 640 --iters 20 2>&1 | tail -1 >> $O/layers.log
  done
done
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "attn_decode or split_decode" > $O/pytest.log 2>&1
echo done > $O/done
