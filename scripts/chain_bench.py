"""Weight-stream rate of the persistent chain kernel, one projection at a time.

    python scripts/chain_bench.py [--model l3|q2] [--T 8 64]

pl_stage_chain_bench launches a chain holding ONE projection of layer 0 (no
dependencies, no finalisation); CUDA events around 20 back-to-back launches give the
per-launch time and the achieved weight GB/s (launch overhead included).
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B, QWEN2_72B  # noqa: E402
from paper_2507_05043_b200 import _native as N  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="l3")
ap.add_argument("--T", type=int, nargs="+", default=[8, 64])
ap.add_argument("--tag", default="")
a = ap.parse_args()
spec = (LLAMA3_8B if a.model == "l3" else QWEN2_72B).with_(num_layers=1)
Tm = max(a.T)
exe = StageExecutor(spec, 0, (0, 1), False, False, torch.device("cuda", 0), max_tokens=Tm, max_reqs=Tm,
                    max_ctx=64, num_blocks=Tm + 4, n_slots=1)
names = ["o", "gate_up", "down", "qkv"]
wbytes = [spec.d * spec.attn_dim * 2, 2 * spec.ffn * spec.d * 2, spec.d * spec.ffn * 2, spec.qkv_dim * spec.d * 2]
st = exe.stream
for T in a.T:
    for kind in range(4):
        N.call("pl_stage_chain_bench", exe.handle, kind, T, 3, st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        N.call("pl_stage_chain_bench", exe.handle, kind, T, 20, st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(json.dumps({"tag": a.tag, "T": T, "proj": names[kind], "us": round(us, 2),
                          "GBps": round(wbytes[kind] / us / 1e3, 1)}), flush=True)
