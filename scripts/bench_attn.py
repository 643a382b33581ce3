"""Prefill attention kernels, mma.sync (FA2) vs tcgen05 (FA4-style): TFLOP/s and agreement.

    python scripts/bench_attn.py [--iters 20]

Causal FLOPs per (head, request of length L) = 4 * hd * L (L + 1) / 2 (QK^T and PV,
the masked upper triangle not counted).  Times are CUDA events around `iters`
back-to-back launches on the current stream after warm-up; the peak is
MEASURED_PEAKS.json's sustained dense bf16 figure.  One JSON line per shape.
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2507_05043_b200 import ops

    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    peak = peaks["bf16_tflops_sustained"]  # a kernel timed inside a long loop
    dev = torch.device("cuda", 0)
    hd = 128
    shapes = [  # (label, lens, Hq, Hkv)
        ("l3-8b 4x2048", [2048] * 4, 32, 8),
        ("l3-8b 16x512", [512] * 16, 32, 8),
        ("l3-8b 1x8192", [8192], 32, 8),
        ("q2-72b 4x2048", [2048] * 4, 64, 8),
        ("bench prefill 64x512", [512] * 64, 32, 8),
        ("mixed lens", [37, 1000, 513, 2048, 5, 1500], 32, 8),
    ]
    for label, lens, Hq, Hkv in shapes:
        T = sum(lens)
        g = torch.Generator(device=dev).manual_seed(T)
        qkv = torch.randn(T, (Hq + 2 * Hkv) * hd, generator=g, device=dev).to(torch.bfloat16)
        cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device=dev)
        flops = sum(4.0 * hd * L * (L + 1) / 2 for L in lens) * Hq
        row = {"shape": label, "lens": lens if len(lens) <= 8 else f"{len(lens)}x{lens[0]}", "Hq": Hq, "Hkv": Hkv}
        outs = {}
        for impl, name in ((1, "mma_sync"), (2, "tcgen05")):
            out = torch.empty(T, Hq * hd, dtype=torch.bfloat16, device=dev)
            for _ in range(3):
                ops.attn_prefill(qkv, cu, max(lens), Hq, Hkv, hd, out=out, impl=impl)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                ops.attn_prefill(qkv, cu, max(lens), Hq, Hkv, hd, out=out, impl=impl)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.iters
            tf = flops / (us * 1e-6) / 1e12
            row[name] = {"us": round(us, 1), "tflops": round(tf, 1),
                         "frac": round(tf / peak, 3) if peak else None}
            outs[name] = out.float()
        d = (outs["mma_sync"] - outs["tcgen05"]).abs()
        row["max_abs_diff"] = round(d.max().item(), 5)
        row["speedup"] = round(row["mma_sync"]["us"] / row["tcgen05"]["us"], 2)
        print(json.dumps(row), flush=True)
    print(json.dumps({"peak_tflops": peak, "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}))


if __name__ == "__main__":
    main()
