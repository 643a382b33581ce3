#!/bin/bash
# tcgen05 prefill attention: parity vs the oracle and the mma.sync kernel, then speed
cd "$(dirname "$0")/.."
O=gpurun_out/attn
mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k attn_prefill -x > $O/pytest.log 2>&1
timeout 300 python scripts/bench_attn.py > $O/bench.log 2>&1
echo done > $O/done
