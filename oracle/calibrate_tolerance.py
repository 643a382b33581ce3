"""ORACLE (test infrastructure): calibrate the GPU-vs-oracle logits tolerance.

SURVEY §8(c)(i): the GPU kernels round at the oracle's bf16 points but sum fp32
products in a different order (tcgen05 k-blocks, split-K partials, attention
splits), and on random-init weights that alone moves logits.  This script
measures how far two bf16-faithful CPU computations drift when they differ
ONLY in fp32 summation order -- the default single pass vs K summed in s fp32
partials added in reversed order (s = 4, 8; oracle/decoder.accumulation_order)
-- through the whole model, for the parity-test workloads:

  tiny   4 layers                      (config 1; tiny-d1024: its d=1024, GQA 8/2 variant)
  l3-32  Llama-3-8B shape, all 32 layers (BASELINE config 2, the benched model)
  q2-10  Qwen2-72B shape, 10 layers (one S=8 stage's depth), qkv bias

Workload per model: 4 requests, hash prompts of 64..112 tokens, 4 continuation
tokens teacher-forced (hash ids), logits at the 4 predicting rows + the last
prompt row.  Output: tests/golden/logit_tolerance.json with the max |dlogit|
(delta), the logit std, and tol = TOL_MULT * delta, which the full-depth GPU
parity tests (tests/test_fullmodel_parity_gpu.py) and bench.py's parity object
apply.  One layer's weights are resident at a time; each layer is generated
once and run under every summation order.

    python -m oracle.calibrate_tolerance [--models tiny,l3-32,q2-10] [--device cpu|cuda]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import decoder as OD  # noqa: E402
from oracle import hashinit as H  # noqa: E402

TOL_MULT = 4.0
ORDERS = (0, 4, 8)
OUT = ROOT / "tests" / "golden" / "logit_tolerance.json"


def models():
    from paper_2507_05043_b200.spec import LLAMA3_8B, QWEN2_72B, TINY

    return {"tiny": TINY, "tiny-d1024": TINY.with_(Hq=8, Hkv=2, d=1024, ffn=1536, vocab=2048),
            "l3-32": LLAMA3_8B, "q2-10": QWEN2_72B.with_(num_layers=10)}


def workload(spec, seed=0, R=4, steps=4):
    seqs, rows = [], []
    for r in range(R):
        L = 64 + 16 * r
        p = torch.from_numpy(H.hash_tokens(L, seed, OD.T_PROMPT + r, spec.vocab))
        gen = torch.from_numpy(H.hash_tokens(steps, seed, 0xABC0 + r, spec.vocab))
        seqs.append(torch.cat([p, gen[:-1]]))
        rows.append(torch.arange(L - 1, L - 1 + steps))
    return seqs, rows


def run(name, spec, device, seed=0):
    o = OD.OracleSpec.from_spec(spec)
    mk = OD.torch_hash_maker(device)
    seqs, rows = workload(o, seed)
    table = OD.rope_table_ref(o.rope_theta, o.hd, 512)
    ids = torch.cat(seqs)
    pos = torch.cat([torch.arange(s.numel()) for s in seqs])
    seg = [s.numel() for s in seqs]
    h0 = OD.make_embed(o, seed, mk)[ids]
    hs = {k: h0 for k in ORDERS}
    e = torch.empty(0, o.Hkv, o.hd, dtype=OD.BF16)
    t0 = time.time()
    for l in range(o.num_layers):
        W = OD.make_layer(o, l, seed, mk)
        for k in ORDERS:
            with OD.accumulation_order(k):
                hs[k] = OD.layer_forward(o, W, hs[k], pos, table, [(e, e) for _ in seqs], seg)
        del W
        print(f"  {name} layer {l + 1}/{o.num_layers} {time.time() - t0:.0f}s", flush=True)
    off = np.concatenate([[0], np.cumsum(seg)[:-1]])
    sel = torch.cat([r + int(b) for r, b in zip(rows, off)])
    fn, lm = OD.make_head(o, seed, mk)
    logits = {}
    for k in ORDERS:
        with OD.accumulation_order(k):
            logits[k] = OD.linear_acc(OD.rmsnorm_ref(hs[k][sel], fn, o.eps), lm)
    delta = max((logits[k] - logits[0]).abs().max().item() for k in ORDERS if k)
    flips = sum(int((logits[k].argmax(-1) != logits[0].argmax(-1)).sum()) for k in ORDERS if k)
    return {"layers": o.num_layers, "d": o.d, "vocab": o.vocab, "rows": int(sel.numel()),
            "logit_std": round(logits[0].std().item(), 5), "delta": round(delta, 6),
            "argmax_flips": flips, "tol_mult": TOL_MULT, "tol": round(TOL_MULT * delta, 6),
            "orders": "single pass vs K in 4 / 8 fp32 partials summed in reversed order"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="tiny,l3-32,q2-10")
    ap.add_argument("--device", default="cpu")
    a = ap.parse_args()
    torch.set_num_threads(os.cpu_count() or 1)
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    ms = models()
    for name in a.models.split(","):
        t = time.time()
        out[name] = run(name, ms[name], a.device)
        out[name]["cpu_s"] = round(time.time() - t, 1)
        print(name, out[name], flush=True)
        OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
