#!/bin/bash
# tcgen05 prefill attention: parity, then item-order / ring-depth variants A/B (experiment builds)
cd "$(dirname "$0")/.."
O=gpurun_out/attn_ab
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
PL_BUILD_VARIANT=ord0 PL_NVCC_EXTRA="-DPL_AT_ORDER=0" python -m paper_2507_05043_b200.build >> $O/build.log 2>&1
PL_BUILD_VARIANT=k2v1 PL_NVCC_EXTRA="-DPL_AT_KST=2 -DPL_AT_VST=1" python -m paper_2507_05043_b200.build >> $O/build.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k attn_prefill > $O/pytest.log 2>&1
timeout 300 python scripts/bench_attn.py > $O/bench_default.log 2>&1
PL_LIB_PATH=paper_2507_05043_b200/_lib_ord0/libb200link.so timeout 300 python scripts/bench_attn.py > $O/bench_ord0.log 2>&1
PL_LIB_PATH=paper_2507_05043_b200/_lib_k2v1/libb200link.so timeout 300 python scripts/bench_attn.py > $O/bench_k2v1.log 2>&1
echo done > $O/done
