#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
PL_CHAIN_VERBOSE=1 PL_CHAIN_TRACE=8 timeout 300 python scripts/chain_trace.py gpurun_out/trace_8.npz > gpurun_out/trace_8.log 2>&1
PL_CHAIN_TRACE=8 timeout 300 python scripts/chain_trace.py gpurun_out/trace_8_T8.npz --T 8 > gpurun_out/trace_8_T8.log 2>&1
for T in 64 16 8 1; do
  echo "T=$T chain=0: $(PL_CHAIN=0 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
  echo "T=$T chain=1: $(PL_CHAIN=1 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
done
timeout 900 python -m pytest tests/test_pipeline_gpu.py -q -x -m gpu -k "decode_logits or config1 or batch_invariant or llama3 or qwen2 or stage_counts" > gpurun_out/pytest_n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_n.log
