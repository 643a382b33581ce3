#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
for R in 8 64; do
  PL_CHAIN=0 timeout 300 python scripts/chain_ab.py /tmp/c0.pt 2 $R > gpurun_out/ab_2_${R}_0.log 2>&1
  PL_CHAIN=1 timeout 300 python scripts/chain_ab.py /tmp/c1.pt 2 $R > gpurun_out/ab_2_${R}_1.log 2>&1
  python - <<PY >> gpurun_out/ab.log 2>&1
import torch
a, b = torch.load("/tmp/c0.pt"), torch.load("/tmp/c1.pt")
print("L=2 R=$R ids equal:", torch.equal(a["ids"], b["ids"]), "max|dhn|:", (a["hn"].float() - b["hn"].float()).abs().max().item(),
      "max|hn|:", a["hn"].float().abs().max().item())
PY
done
for k in 7 8; do
  PL_CHAIN_VERBOSE=1 PL_CHAIN_TRACE=$k timeout 300 python scripts/chain_trace.py gpurun_out/trace_$k.npz > gpurun_out/trace_$k.log 2>&1
done
for T in 64 16 8 1; do
  echo "T=$T chain=0: $(PL_CHAIN=0 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
  echo "T=$T chain=1: $(PL_CHAIN=1 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
done
timeout 900 python -m pytest tests/test_pipeline_gpu.py -q -x -m gpu > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_e.log
