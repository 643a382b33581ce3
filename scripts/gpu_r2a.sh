#!/bin/bash
# round 2, first GPU pass: chain kernel A/B, decode layer timing, parity tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
for L in 2; do for R in 8 64; do
  PL_CHAIN=0 timeout 300 python scripts/chain_ab.py /tmp/c0.pt $L $R > gpurun_out/ab_${L}_${R}_0.log 2>&1
  PL_CHAIN=1 timeout 300 python scripts/chain_ab.py /tmp/c1.pt $L $R > gpurun_out/ab_${L}_${R}_1.log 2>&1
  python - <<PY >> gpurun_out/ab.log 2>&1
import torch
a, b = torch.load("/tmp/c0.pt"), torch.load("/tmp/c1.pt")
print("L=$L R=$R ids equal:", torch.equal(a["ids"], b["ids"]), "max|dhn|:", (a["hn"].float() - b["hn"].float()).abs().max().item(),
      "max|hn|:", a["hn"].float().abs().max().item())
PY
done; done
for T in 64 16 8 1; do
  echo "T=$T chain=0: $(PL_CHAIN=0 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
  echo "T=$T chain=1: $(PL_CHAIN=1 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
done
timeout 1500 python -m pytest tests/test_pipeline_gpu.py tests/test_kernels_gpu.py tests/test_fullmodel_parity_gpu.py -q -s -m gpu > gpurun_out/pytest_a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_a.log
