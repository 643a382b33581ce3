#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
for R in 16 33 64; do
  PL_CHAIN=0 timeout 300 python scripts/chain_ab.py /tmp/c0.pt 2 $R > /dev/null 2>&1
  PL_CHAIN=1 timeout 300 python scripts/chain_ab.py /tmp/c1.pt 2 $R > gpurun_out/abf_$R.log 2>&1
  python - <<PY >> gpurun_out/abf.log 2>&1
import torch
a, b = torch.load("/tmp/c0.pt"), torch.load("/tmp/c1.pt")
d = (a["hn"].float() - b["hn"].float()).abs()   # [steps, R, d]
print("R=$R per step max:", [round(x, 4) for x in d.amax(dim=(1, 2)).tolist()])
print("  step-1 per request max:", [round(x, 3) for x in d[1].amax(dim=1).tolist()])
bad = (d[1] > 0.5).nonzero()
print("  bad (req, feature) at step 1 (first 20):", bad[:20].tolist(), "count", bad.shape[0])
PY
done
