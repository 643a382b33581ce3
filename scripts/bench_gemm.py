"""Micro-benchmark of the decode GEMMs / attention at model shapes (CUDA events).

    python scripts/bench_gemm.py [--T 64] [--model l3|q2]

Weights rotate over enough copies to exceed the 126 MB L2, so every call
streams its weights from HBM.  Prints one JSON line per kernel with the
average launch time and achieved GB/s of algorithmic bytes.
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B, QWEN2_72B, ops  # noqa: E402


def timeit(fn, iters=40, warm=3):
    """Device time per call: the calls are captured into one CUDA graph and replayed,
    so host (Python/ctypes) launch overhead is excluded."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(warm):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, nargs="+", default=[8, 16, 32, 64])
    ap.add_argument("--model", default="l3")
    ap.add_argument("--shapes", nargs="*", default=None,
                    help="custom N,K pairs (plain store epilogue), e.g. 18944,4096 18944,1024")
    ap.add_argument("--packed", action="store_true", help="pre-swizzled weights (pl_pack_weight), as served")
    a = ap.parse_args()
    spec = {"l3": LLAMA3_8B, "q2": QWEN2_72B}[a.model]
    dev = torch.device("cuda", 0)
    shapes = {"qkv": (spec.qkv_dim, spec.d, ops.EPI_NONE), "o": (spec.d, spec.attn_dim, ops.EPI_RESIDUAL),
              "gate_up": (2 * spec.ffn, spec.d, ops.EPI_SWIGLU), "down": (spec.d, spec.ffn, ops.EPI_RESIDUAL),
              "lm_head": (spec.vocab, spec.d, ops.EPI_ARGMAX)}
    if a.shapes:
        shapes = {f"N{n}K{k}": (int(n), int(k), ops.EPI_NONE) for n, k in (x.split(",") for x in a.shapes)}
    for name, (N, K, epi) in shapes.items():
        wbytes = N * K * 2
        copies = max(1, -(-300_000_000 // wbytes))
        ws = [torch.randn(N, K, device=dev).to(torch.bfloat16) * 0.02 for _ in range(copies)]
        gemm = ops.gemm
        if a.packed and N % 256 == 0:
            ws = [ops.pack_weight(w, interleave=epi == ops.EPI_SWIGLU) for w in ws]
            gemm = ops.gemm_packed
        for T in a.T:
            if epi == ops.EPI_ARGMAX and T > 256:
                continue
            x = torch.randn(T, K, device=dev).to(torch.bfloat16)
            res = torch.randn(T, N, device=dev).to(torch.bfloat16) if epi == ops.EPI_RESIDUAL else None
            out = torch.empty(T, N // 2 if epi == ops.EPI_SWIGLU else N, device=dev, dtype=torch.bfloat16)

            def fn(i):
                if epi == ops.EPI_RESIDUAL:
                    gemm(x, ws[i % copies], epi, residual=res, out=res)
                elif epi == ops.EPI_ARGMAX:
                    gemm(x, ws[i % copies], epi)
                else:
                    gemm(x, ws[i % copies], epi, out=out)

            us = timeit(fn)
            print(json.dumps({"kernel": name, "T": T, "N": N, "K": K, "packed": gemm is not ops.gemm, "us": round(us, 2),
                              "GBps": round(wbytes / us / 1e3, 1)}), flush=True)
        del ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
