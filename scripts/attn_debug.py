"""Run one prefill-attention case per process (a fault poisons the context):
    python scripts/attn_debug.py IMPL HQ HKV L1,L2,...   -> prints max error vs the oracle"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    from oracle import decoder as OD
    from paper_2507_05043_b200 import ops

    impl, Hq, Hkv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    lens = [int(x) for x in sys.argv[4].split(",")]
    hd, T = 128, sum(lens)
    g = torch.Generator().manual_seed(T + Hq)
    qkv = torch.randn(T, (Hq + 2 * Hkv) * hd, generator=g).to(torch.bfloat16)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    out = ops.attn_prefill(qkv.cuda(), cu.cuda(), max(lens), Hq, Hkv, hd, impl=impl).float().cpu()
    x = qkv.reshape(T, Hq + 2 * Hkv, hd)
    ref = torch.cat([OD.attention_ref(x[s:s + n, :Hq], x[s:s + n, Hq:Hq + Hkv], x[s:s + n, Hq + Hkv:], 0)
                     for s, n in zip(cu[:-1].tolist(), lens)]).float()
    err = (out - ref).abs()
    rows = err.reshape(T, -1).amax(1)
    bad = (rows > 0.05).nonzero().flatten().tolist()
    print(f"impl {impl} Hq {Hq} Hkv {Hkv} lens {lens}: max err {err.max().item():.4g}; bad rows {bad[:20]}"
          f"{'...' if len(bad) > 20 else ''} ({len(bad)})", flush=True)


if __name__ == "__main__":
    main()
