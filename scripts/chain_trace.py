"""Timeline of one persistent chain launch (debug; PL_CHAIN_TRACE=<launch number>).

    PL_CHAIN_TRACE=8 python scripts/chain_trace.py out.npz [--T 64] [--layers 2]

Runs decode forwards of a truncated Llama-3-8B-shape stage (each forward launches
chains 1 + layers: qkv-only, then one per layer), then saves the per-unit stamps of
the traced launch and prints a summary.
"""

import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B  # noqa: E402
from paper_2507_05043_b200 import _native as N  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402
from paper_2507_05043_b200.profiler import time_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--T", type=int, default=64)
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--ctx", type=int, default=640)
a = ap.parse_args()
spec = LLAMA3_8B.with_(num_layers=a.layers)
exe = StageExecutor(spec, 0, (0, a.layers), True, False, torch.device("cuda", 0), max_tokens=a.T,
                    max_reqs=a.T, max_ctx=a.ctx + 1, num_blocks=a.T * (-(-(a.ctx + 1) // 64)) + 64, n_slots=1)
for _ in range(4):
    t = time_forward(exe, a.T, True, ctx=a.ctx, reps=1)
print(f"forward {t * 1e6:.1f} us")
buf = np.zeros(4 * 148 * 64 * 4, dtype=np.uint64)  # up to 4 CTAs per SM
grid = C.c_int32()
N.call("pl_stage_chain_trace", exe.handle, buf.ctypes.data, buf.size, C.byref(grid))
g = grid.value
tr = buf[: g * 64 * 4].reshape(g, 64, 4)
M40 = (1 << 40) - 1
claim_t = tr[:, :, 0] & M40
claim_i = (tr[:, :, 0] >> 40).astype(np.int64)
valid = tr[:, :, 0] > 0
t0 = int(claim_t[valid].min())
rel = lambda x: (((x.astype(np.int64) & M40) - t0 + (1 << 39)) % (1 << 40) - (1 << 39)) / 1e3  # noqa: E731
np.savez(a.out, claim_t=rel(claim_t), claim_i=claim_i, pop=rel(tr[:, :, 1]), ready=rel(tr[:, :, 2]),
         done=rel(tr[:, :, 3]), valid=valid)
units = valid.sum(1)
end = np.where(valid, rel(tr[:, :, 3]), 0).max(1)
print(f"units per CTA: min {units.min()} max {units.max()} mean {units.mean():.2f}")
print(f"CTA end (us): min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f}")
epi = np.where(valid, rel(tr[:, :, 3]) - rel(tr[:, :, 2]), np.nan)
wait = np.where(valid, rel(tr[:, :, 2]) - rel(tr[:, :, 1]), np.nan)
print(f"epilogue us: median {np.nanmedian(epi):.2f} p90 {np.nanpercentile(epi, 90):.2f} max {np.nanmax(epi):.2f}")
print(f"pop->ready us: median {np.nanmedian(wait):.2f} p90 {np.nanpercentile(wait, 90):.2f} max {np.nanmax(wait):.2f}")
slow = np.argsort(-end)[:3]
for c in slow:
    print(f"CTA {c}: " + "; ".join(
        f"#{claim_i[c, k]} claim {rel(claim_t[c, k:k+1])[0]:.1f} pop {rel(tr[c, k:k+1, 1])[0]:.1f} "
        f"ready {rel(tr[c, k:k+1, 2])[0]:.1f} done {rel(tr[c, k:k+1, 3])[0]:.1f}" for k in range(units[c])))
