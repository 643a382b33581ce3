"""Profiling driver: decode (and optionally prefill) forwards of a truncated
Llama-3-8B-shape stage, for ncu captures of the hot kernels.

    python scripts/profile_decode.py [--layers 2] [--T 64] [--ctx 640] [--iters 5] [--prefill 0]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402
from paper_2507_05043_b200.profiler import time_forward  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--T", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=640)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--prefill", type=int, default=0)
    ap.add_argument("--last", type=int, default=1)
    a = ap.parse_args()
    spec = LLAMA3_8B.with_(num_layers=a.layers)
    max_tokens = max(a.T, a.prefill)
    exe = StageExecutor(spec, 0, (0, a.layers), True, bool(a.last), torch.device("cuda", 0),
                        max_tokens=max_tokens, max_reqs=max(a.T, 1), max_ctx=max(a.ctx, a.prefill) + 1,
                        num_blocks=a.T * (-(-(a.ctx + 1) // 64)) + 64, n_slots=1)
    for _ in range(a.iters):
        t = time_forward(exe, a.T, True, ctx=a.ctx, reps=1)
    print(f"decode T={a.T} ctx={a.ctx}: {t * 1e6:.1f} us per {a.layers}-layer forward")
    if a.prefill:
        t = time_forward(exe, a.prefill, False, reps=1)
        print(f"prefill T={a.prefill}: {t * 1e3:.3f} ms per {a.layers}-layer forward")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
