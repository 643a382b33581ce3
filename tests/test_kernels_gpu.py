"""Kernel parity: every libb200link kernel vs the CPU oracle (oracle/decoder.py).

Tolerances (stated per test):
* integer / byte work (hash init, embedding gather, argmax outside the tie
  band, RoPE+KV append) is bit-exact;
* bf16 outputs of fp32 reductions (RMSNorm, GEMM epilogues, attention) may
  differ from the oracle only by the fp32 summation order, i.e. at most a
  couple of bf16 ulps: |gpu - ref| <= 2^-7 |ref| + atol.
"""

import math

import numpy as np
import pytest
import torch

from oracle import decoder as OD
from oracle import hashinit as H

pytestmark = pytest.mark.gpu

BF16 = torch.bfloat16


@pytest.fixture(scope="module")
def ops():
    from paper_2507_05043_b200 import ops as O

    return O


def dev():
    return torch.device("cuda:0")


def close_bf16(gpu, ref, rel=2.0 ** -7, atol=1e-3, scale=None):
    """|gpu - ref| <= rel * scale + atol, scale = |ref| unless the op sums terms that
    can cancel (residual adds: scale = |a| + |b| of the two rounded addends)."""
    g = gpu.float().cpu()
    r = ref.float().cpu()
    err = (g - r).abs()
    bound = rel * (r.abs() if scale is None else scale) + atol
    bad = (err > bound).sum().item()
    assert bad == 0, f"{bad} / {err.numel()} elements out of tolerance; max err {err.max().item():.3g}"


@pytest.mark.parametrize("n,tid,scale,offset", [(1, 3, 1.0, 0.0), (1000, 7, 0.0346, 0.0),
                                                 (1 << 20, 0xFFFF0001, 0.02, 0.0),
                                                 (4097, 17, 0.05, 1.0)])
def test_fill_hash_bit_exact(ops, n, tid, scale, offset):
    t = torch.empty(n, dtype=BF16, device=dev())
    ops.fill_hash_(t, 0, tid, scale, offset)
    want = H.hash_bf16_bits(n, 0, tid, scale, offset)
    got = t.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want)


def test_embed_exact(ops):
    table = torch.randn(512, 256).to(BF16)
    ids = torch.randint(0, 512, (37,))
    out = ops.embed(ids.to(dev()), table.to(dev()))
    assert torch.equal(out.cpu(), table[ids])
    # decode path: gather through the per-slot feedback table
    last = torch.randint(0, 512, (16,))
    slot = torch.randint(0, 16, (9,), dtype=torch.int32)
    out = ops.embed(None, table.to(dev()), req_slot=slot.to(dev()), last_token=last.to(dev()))
    assert torch.equal(out.cpu(), table[last[slot.long()]])


@pytest.mark.parametrize("rows,d", [(1, 256), (7, 4096), (64, 8192), (300, 4096)])
def test_rmsnorm(ops, rows, d):
    g = torch.Generator().manual_seed(rows * 7 + d)
    x = (torch.randn(rows, d, generator=g) * 3).to(BF16)
    w = (1 + 0.05 * torch.randn(d, generator=g)).to(BF16)
    out = ops.rmsnorm(x.to(dev()), w.to(dev()), 1e-5)
    close_bf16(out, OD.rmsnorm_ref(x, w, 1e-5), rel=2.0 ** -7, atol=1e-6)


def test_rmsnorm_row_gather(ops):
    x = torch.randn(50, 256).to(BF16)
    w = torch.ones(256).to(BF16)
    idx = torch.tensor([49, 0, 17], dtype=torch.int32)
    out = ops.rmsnorm(x.to(dev()), w.to(dev()), 1e-6, row_idx=idx.to(dev()))
    close_bf16(out, OD.rmsnorm_ref(x[idx.long()], w, 1e-6), atol=1e-6)


GEMM_SHAPES = [  # (T, N, K)
    (1, 512, 256), (5, 640, 256), (16, 6144, 4096), (17, 384, 768), (64, 4096, 4096),
    (100, 1024, 512), (256, 512, 256), (300, 512, 256), (1000, 1536, 256), (2048, 768, 1024),
    # more weight tiles than SMs (148 < N/128 < 296): two waves of persistent CTAs
    (64, 28672, 4096), (7, 20480, 1024), (130, 19200, 512),
]


@pytest.mark.parametrize("T,N,K", GEMM_SHAPES)
def test_gemm_store(ops, T, N, K):
    g = torch.Generator().manual_seed(T * 31 + N + K)
    x = torch.randn(T, K, generator=g).to(BF16)
    w = (torch.randn(N, K, generator=g) * 0.05).to(BF16)
    out = ops.gemm(x.to(dev()), w.to(dev()))
    close_bf16(out, OD.linear_acc(x, w), atol=1e-3)


@pytest.mark.parametrize("T,N,K", [(3, 512, 256), (64, 6144, 4096), (700, 512, 256)])
def test_gemm_bias(ops, T, N, K):
    g = torch.Generator().manual_seed(5)
    x = torch.randn(T, K, generator=g).to(BF16)
    w = (torch.randn(N, K, generator=g) * 0.05).to(BF16)
    b = torch.randn(N, generator=g).to(BF16)
    out = ops.gemm(x.to(dev()), w.to(dev()), ops.EPI_BIAS, bias=b.to(dev()))
    close_bf16(out, OD.linear_acc(x, w) + b.float(), atol=1e-3)


@pytest.mark.parametrize("T,N,K", [(8, 256, 256), (64, 4096, 14336), (513, 256, 768)])
def test_gemm_residual_inplace(ops, T, N, K):
    g = torch.Generator().manual_seed(9)
    x = torch.randn(T, K, generator=g).to(BF16)
    w = (torch.randn(N, K, generator=g) * 0.02).to(BF16)
    h = torch.randn(T, N, generator=g).to(BF16)
    hd = h.to(dev())
    ops.gemm(x.to(dev()), w.to(dev()), ops.EPI_RESIDUAL, residual=hd, out=hd)
    acc = OD.rbf(OD.linear_acc(x, w))
    ref = acc + h.float()
    close_bf16(hd, ref, rel=2.0 ** -6, atol=1e-3, scale=acc.abs() + h.float().abs())  # two roundings


@pytest.mark.parametrize("T,ffn,K", [(4, 768, 256), (32, 14336, 4096), (400, 768, 256)])
def test_gemm_swiglu(ops, T, ffn, K):
    g = torch.Generator().manual_seed(11)
    x = torch.randn(T, K, generator=g).to(BF16)
    w = (torch.randn(2 * ffn, K, generator=g) * 0.05).to(BF16)
    out = ops.gemm(x.to(dev()), w.to(dev()), ops.EPI_SWIGLU)
    wg, wu = OD.deinterleave_gate_up(w)
    g_acc, u_acc = OD.linear_acc(x, wg), OD.linear_acc(x, wu)
    ref = OD.swiglu_ref(g_acc, u_acc)
    # a 1-ulp flip of bf16(g) from the fp32 summation order moves silu(g)*u by up to
    # ~ulp(g) * |u| (silu' <= 1.1): bound relative to |ref| + |g*u|
    scale = ref.float().abs() + (OD.rbf(g_acc) * OD.rbf(u_acc)).abs()
    close_bf16(out, ref, rel=2.0 ** -6, atol=2e-3, scale=scale)


@pytest.mark.parametrize("R,V,d", [(1, 512, 256), (8, 128256, 4096), (64, 32000, 256), (200, 1000, 256)])
def test_lmhead_argmax(ops, R, V, d):
    g = torch.Generator().manual_seed(R + V)
    h = torch.randn(R, d, generator=g).to(BF16)
    w = (torch.randn(V, d, generator=g) * 0.05).to(BF16)
    ids = ops.lmhead_argmax(h.to(dev()), w.to(dev())).cpu()
    logits = OD.linear_acc(h, w)
    top2 = logits.topk(2, dim=-1).values
    tie = (top2[:, 0] - top2[:, 1]) < 1e-3 * top2[:, 0].abs().clamp(min=1)
    ref = logits.argmax(-1)
    ok = (ids == ref) | tie
    assert ok.all(), f"argmax mismatch outside tie band at rows {torch.nonzero(~ok).flatten().tolist()}"
    # chosen id must be (near-)maximal
    assert (logits.gather(1, ids[:, None]).squeeze(1) >= top2[:, 0] - 1e-3 * top2[:, 0].abs().clamp(min=1)).all()


def test_rope_kv_bit_exact(ops):
    T, Hq, Hkv, hd = 70, 4, 2, 128
    g = torch.Generator().manual_seed(3)
    qkv = torch.randn(T, (Hq + 2 * Hkv) * hd, generator=g).to(BF16)
    pos = torch.randint(0, 900, (T,), dtype=torch.int32)
    table = OD.rope_table_ref(5e5, hd, 1024)
    num_blocks = 8
    slot = torch.randperm(num_blocks * 64)[:T].to(torch.int32)
    kc = torch.zeros(num_blocks, Hkv, 64, hd, dtype=BF16, device=dev())
    vc = torch.zeros_like(kc)
    q_gpu = qkv.to(dev())
    ops.rope_kv_write(q_gpu, pos.to(dev()), slot.to(dev()), table.to(dev()), kc, vc, Hq, Hkv, hd)
    x = qkv.reshape(T, Hq + 2 * Hkv, hd)
    ref_q = OD.rope_ref(x[:, :Hq], pos, table)
    ref_k = OD.rope_ref(x[:, Hq:Hq + Hkv], pos, table)
    got = q_gpu.cpu().reshape(T, Hq + 2 * Hkv, hd)
    assert torch.equal(got[:, :Hq], ref_q)
    assert torch.equal(got[:, Hq:Hq + Hkv], ref_k)
    assert torch.equal(got[:, Hq + Hkv:], x[:, Hq + Hkv:])
    kc, vc = kc.cpu(), vc.cpu()
    for t in range(T):
        b, o = int(slot[t]) // 64, int(slot[t]) % 64
        assert torch.equal(kc[b, :, o], ref_k[t])
        assert torch.equal(vc[b, :, o], x[t, Hq + Hkv:])


@pytest.mark.parametrize("impl", [1, 2], ids=["mma_sync", "tcgen05"])
@pytest.mark.parametrize("lens,Hq,Hkv", [([128] * 8, 2, 1), ([1, 63, 64, 65, 200], 4, 2),
                                         ([512, 512], 32, 8), ([2048], 8, 1), ([300, 1, 129, 700], 8, 8),
                                         ([1000, 24], 64, 8)])
def test_attn_prefill(ops, lens, Hq, Hkv, impl):
    hd = 128
    T = sum(lens)
    g = torch.Generator().manual_seed(sum(lens) + Hq)
    qkv = torch.randn(T, (Hq + 2 * Hkv) * hd, generator=g).to(BF16)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    out = ops.attn_prefill(qkv.to(dev()), cu.to(dev()), max(lens), Hq, Hkv, hd, impl=impl).cpu()
    x = qkv.reshape(T, Hq + 2 * Hkv, hd)
    refs = []
    for r, n in enumerate(lens):
        s = int(cu[r])
        refs.append(OD.attention_ref(x[s:s + n, :Hq], x[s:s + n, Hq:Hq + Hkv], x[s:s + n, Hq + Hkv:], 0))
    close_bf16(out, torch.cat(refs), rel=2.0 ** -6, atol=4e-3)


@pytest.mark.parametrize("ctx,Hq,Hkv", [([1, 5, 64, 65, 640], 32, 8), ([700, 1300], 8, 8),
                                        ([129] * 16, 2, 1), ([3000], 64, 8)])
def test_attn_decode_paged(ops, ctx, Hq, Hkv):
    hd, bs = 128, 64
    R = len(ctx)
    g = torch.Generator().manual_seed(sum(ctx) + Hq)
    max_blocks = max((c + bs - 1) // bs for c in ctx)
    num_blocks = R * max_blocks + 3
    perm = torch.randperm(num_blocks, generator=g)
    bt = perm[: R * max_blocks].reshape(R, max_blocks).to(torch.int32)
    kc = torch.randn(num_blocks, Hkv, bs, hd, generator=g).to(BF16)
    vc = torch.randn(num_blocks, Hkv, bs, hd, generator=g).to(BF16)
    q = torch.randn(R, Hq * hd, generator=g).to(BF16)
    ctx_t = torch.tensor(ctx, dtype=torch.int32)
    out = ops.attn_decode(q.to(dev()), kc.to(dev()), vc.to(dev()), bt.to(dev()), ctx_t.to(dev()),
                          max(ctx), Hq, Hkv, hd).cpu()
    refs = []
    for r in range(R):
        pages = bt[r, : (ctx[r] + bs - 1) // bs].long()
        k = kc[pages].permute(0, 2, 1, 3).reshape(-1, Hkv, hd)[: ctx[r]]
        v = vc[pages].permute(0, 2, 1, 3).reshape(-1, Hkv, hd)[: ctx[r]]
        refs.append(OD.attention_ref(q[r].reshape(1, Hq, hd), k, v, None))
    # P is rounded to bf16 for the tensor-core P.V (as in the prefill kernel)
    close_bf16(out, torch.cat(refs), rel=2.0 ** -6, atol=4e-3)


def _paged_case(ctx, Hq, Hkv, seed, hd=128, bs=64):
    R = len(ctx)
    g = torch.Generator().manual_seed(seed)
    max_blocks = max((c + bs - 1) // bs for c in ctx)
    num_blocks = R * max_blocks + 3
    perm = torch.randperm(num_blocks, generator=g)
    bt = perm[: R * max_blocks].reshape(R, max_blocks).to(torch.int32)
    kc = torch.randn(num_blocks, Hkv, bs, hd, generator=g).to(BF16)
    vc = torch.randn(num_blocks, Hkv, bs, hd, generator=g).to(BF16)
    q = torch.randn(R, Hq * hd, generator=g).to(BF16)
    refs = []
    for r in range(R):
        pages = bt[r, : (ctx[r] + bs - 1) // bs].long()
        k = kc[pages].permute(0, 2, 1, 3).reshape(-1, Hkv, hd)[: ctx[r]]
        v = vc[pages].permute(0, 2, 1, 3).reshape(-1, Hkv, hd)[: ctx[r]]
        refs.append(OD.attention_ref(q[r].reshape(1, Hq, hd), k, v, None))
    return q, kc, vc, bt, torch.tensor(ctx, dtype=torch.int32), torch.cat(refs)


def test_split_decode_shared_workspace_across_shapes(ops):
    """One workspace (sized for the largest launch, as a stage sizes it) serves split
    launches of different R and context: R=1 at a long context, then R=16, then R=1
    again.  The arrival counters sit at fixed addresses at the end of the workspace, so
    no launch's partials land on another launch's counters (attention.cu)."""
    Hq, Hkv, hd = 32, 8, 128
    from paper_2507_05043_b200 import _native as NN

    ws_bytes = NN.lib().pl_attn_decode_workspace_bytes(16, Hq, 4096, hd)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev())
    cases = [[4000], [1100 + 37 * i for i in range(16)], [3000], [1500] * 16]
    for i, ctx in enumerate(cases):
        q, kc, vc, bt, ctx_t, ref = _paged_case(ctx, Hq, Hkv, seed=100 + i)
        out = ops.attn_decode(q.to(dev()), kc.to(dev()), vc.to(dev()), bt.to(dev()), ctx_t.to(dev()),
                              max(ctx), Hq, Hkv, hd, ws=ws).cpu()
        close_bf16(out, ref, rel=2.0 ** -6, atol=4e-3)
    # every counter is back to zero
    tail = ws[ws_bytes - 16 * Hkv * 4:].view(torch.int32)
    assert int(tail.abs().sum()) == 0


_PAIR_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_2507_05043_b200 import ops
d = torch.device("cuda:0")
outs = []
for (T, Nw, K, epi) in {cases!r}:
    g = torch.Generator().manual_seed(T + Nw + K + epi)
    x = torch.randn(T, K, generator=g).to(torch.bfloat16).to(d)
    w = (torch.randn(Nw, K, generator=g) * 0.05).to(torch.bfloat16).to(d)
    b = torch.randn(Nw, generator=g).to(torch.bfloat16).to(d)
    h = torch.randn(T, Nw, generator=g).to(torch.bfloat16).to(d)
    if epi == ops.EPI_RESIDUAL:
        ops.gemm(x, w, epi, residual=h, out=h)
        outs.append(h.cpu())
    else:
        outs.append(ops.gemm(x, w, epi, bias=b if epi == ops.EPI_BIAS else None).cpu())
torch.cuda.synchronize()
torch.save(outs, sys.argv[1])
"""


def test_gemm_pair_bit_identical(tmp_path):
    """Prefill GEMMs on CTA pairs (tcgen05.mma.cta_group::2, 256 x 256 tiles) vs the
    single-CTA kernel (M = 128): same k order per output element -> bit-identical,
    for every prefill epilogue and ragged T (packed weights through the pair kernel's
    3-D TMA box: test_pipeline_gpu.py::test_packed_weights_bit_identical at T = 600)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    from paper_2507_05043_b200 import ops as O

    root = str(Path(__file__).resolve().parent.parent)
    cases = [(300, 512, 256, O.EPI_NONE), (1000, 1536, 256, O.EPI_NONE), (700, 512, 256, O.EPI_BIAS),
             (513, 256, 768, O.EPI_RESIDUAL), (777, 1536, 512, O.EPI_SWIGLU), (2048, 6144, 4096, O.EPI_NONE),
             (4096, 4096, 4096, O.EPI_RESIDUAL), (5000, 2048, 1024, O.EPI_SWIGLU)]
    script = tmp_path / "pair.py"
    script.write_text(_PAIR_SCRIPT.format(root=root, cases=cases))
    res = []
    for pair in ("0", "1"):
        out = tmp_path / f"o{pair}.pt"
        env = dict(os.environ, PL_GEMM_PAIR=pair)
        p = subprocess.run([sys.executable, str(script), str(out)], env=env, capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
        res.append(torch.load(out))
    for c, a, b in zip(cases, *res):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16)), f"case {c}: pair != single-CTA"


@pytest.mark.parametrize("T,R", [(64, 4), (16, 16), (200, 8)])
def test_cluster_splitk_bit_identical(tmp_path, T, R):
    """Cluster split-K (partials reduced over DSMEM inside the GEMM, QKV+RoPE+KV append
    in the cluster epilogue) vs partials + reduce kernels: a prefill and three decode
    steps of a 2-layer Llama-3-shape stage are bit-identical (hidden states and ids)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    script = Path(__file__).resolve().parent / "_stage_steps.py"
    res = []
    for csk in ("0", "7"):
        out = tmp_path / f"s{csk}.pt"
        p = subprocess.run([sys.executable, str(script), str(out), str(T), str(R)],
                           env=dict(os.environ, PL_CSK=csk), capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
        res.append(torch.load(out))
    for i, (a, b) in enumerate(zip(*res)):
        if a.dtype == torch.bfloat16:
            a, b = a.view(torch.int16), b.view(torch.int16)
        assert torch.equal(a, b), f"output {i} differs between PL_CSK=0 and 7"


@pytest.mark.parametrize("T,N,K,epi", [(16, 6144, 4096, 0), (64, 4096, 4096, 3), (64, 2048, 1024, 2),
                                       (8, 128256 // 256 * 256, 256, 4), (300, 1024, 512, 1), (600, 1536, 512, 2)])
def test_gemm_packed_bit_identical(ops, T, N, K, epi):
    """pl_gemm_packed on pl_pack_weight tiles == pl_gemm on the row-major weight (decode
    split-K / cluster paths, argmax, prefill single-CTA and CTA-pair paths)."""
    g = torch.Generator().manual_seed(T + N + K + epi)
    x = torch.randn(T, K, generator=g).to(BF16).to(dev())
    w = (torch.randn(N, K, generator=g) * 0.05).to(BF16).to(dev())
    b = torch.randn(N, generator=g).to(BF16).to(dev())
    h = torch.randn(T, N, generator=g).to(BF16).to(dev())
    wp = ops.pack_weight(w, interleave=epi == ops.EPI_SWIGLU)
    if epi == ops.EPI_RESIDUAL:
        h2 = h.clone()
        ops.gemm(x, w, epi, residual=h, out=h)
        ops.gemm_packed(x, wp, epi, residual=h2, out=h2)
        a, c = h, h2
    else:
        kw = {"bias": b} if epi == ops.EPI_BIAS else {}
        a = ops.gemm(x, w, epi, **kw)
        c = ops.gemm_packed(x, wp, epi, **kw)
    torch.cuda.synchronize()
    if a.dtype == BF16:
        a, c = a.view(torch.int16), c.view(torch.int16)
    assert torch.equal(a.cpu(), c.cpu())


_PPS_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
from test_kernels_gpu import _paged_case
from paper_2507_05043_b200 import ops
d = torch.device("cuda:0")
outs = []
for i, (ctx, Hq, Hkv) in enumerate({cases!r}):
    q, kc, vc, bt, ctx_t, ref = _paged_case(ctx, Hq, Hkv, seed=7 + i)
    out = ops.attn_decode(q.to(d), kc.to(d), vc.to(d), bt.to(d), ctx_t.to(d), max(ctx), Hq, Hkv, 128).cpu()
    outs.append((out, ref))
torch.save(outs, sys.argv[1])
"""


@pytest.mark.parametrize("pps", ["1", "3", "32"])
def test_attn_decode_pages_per_split_override(tmp_path, pps):
    """PL_ATTN_PPS (pages per decode-attention split; default 16) at its extremes: one page
    per split (up to 47 splits merged by the last arriver), an odd split, and 32 (every
    block-table entry of a split travels in one warp-wide load)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    cases = [([3000], 32, 8), ([65, 640, 1300, 2047], 8, 2), ([129] * 8, 64, 8)]
    script = tmp_path / "pps.py"
    script.write_text(_PPS_SCRIPT.format(root=str(root), tests=str(root / "tests"), cases=cases))
    out = tmp_path / "pps.pt"
    p = subprocess.run([sys.executable, str(script), str(out)], env=dict(os.environ, PL_ATTN_PPS=pps),
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    for got, ref in torch.load(out):
        close_bf16(got, ref, rel=2.0 ** -6, atol=4e-3)
