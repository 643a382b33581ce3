#!/bin/bash
# round 2: dynamic-claim chain kernel -- A/B numerics, layer timing, launch list
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
for T in 64 16 1; do
  echo "T=$T chain=0: $(PL_CHAIN=0 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
  echo "T=$T chain=1: $(PL_CHAIN=1 timeout 300 python scripts/profile_decode.py --layers 4 --T $T --iters 5 --last 0 2>&1 | tail -1)" >> gpurun_out/layer.log
done
PL_CHAIN=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_chain.csv \
  python scripts/profile_decode.py --layers 4 --T 64 --iters 2 --last 0 > gpurun_out/ncu_chain.log 2>&1
timeout 900 python -m pytest tests/test_fullmodel_parity_gpu.py tests/test_pipeline_gpu.py -q -s -m gpu > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_b.log
