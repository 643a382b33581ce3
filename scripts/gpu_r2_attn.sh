#!/bin/bash
# tcgen05 prefill attention: parity vs the oracle and the mma.sync kernel, then speed
cd "$(dirname "$0")/.."
O=gpurun_out/attn
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
for c in "2 1 256" "2 1 200" "4 2 1,63,64,65,200" "8 1 256" "32 8 512" "2 1 1000"; do
  timeout 60 python scripts/attn_debug.py 2 $c >> $O/cases.log 2>&1 || echo "FAILED: $c" >> $O/cases.log
done
grep -q FAILED $O/cases.log && { echo done > $O/done; exit 0; }
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k attn_prefill > $O/pytest.log 2>&1
timeout 300 python scripts/bench_attn.py > $O/bench.log 2>&1
echo done > $O/done
