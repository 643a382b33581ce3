"""ORACLE (test infrastructure only): CPU restatement of the per-stage decoder forward.

The reference replaces this computation with a latency-table lookup
(`compute_time`, pipelink/engine.py:384, profiles.py:95-121); in MoLink it is
vLLM's Llama/Qwen2 forward, with no pinned version.  So this
oracle follows the public architecture definitions in the image's
transformers 5.5.0 (outside /root/reference):

  RMSNorm        modeling_llama.py:62-67   fp32 math, cast to bf16 BEFORE the weight multiply
  RoPE           modeling_llama.py:111-135 cos/sin in fp32 then bf16; :138-168 rotate_half,
                                            every tensor op rounded to bf16
  MLP            modeling_llama.py:182-184 down(act(gate(x)) * up(x)), each op rounded to bf16
  attention      modeling_llama.py:209-221 softmax in fp32 (here: scores and P.V in fp32)
  decoder layer  modeling_llama.py:313-331 residual adds in bf16
  Qwen2 bias     modeling_qwen2.py:200-203 q/k/v bias
  greedy next token = argmax of fp32 logits at each request's last position.

Linear layers accumulate in fp32 (bf16 inputs are exact in fp32).  The GPU
kernels round at the same points; only the fp32 summation order differs, which
is what the stated logits tolerance covers.  Weights and prompts come from
oracle/hashinit.py (bit-identical to the GPU fill).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU baseline use this module.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import hashinit as H

BF16 = torch.bfloat16

# tensor-id contract (paper_2507_05043_b200/spec.py)
T_ATTN_NORM, T_QKV, T_QKV_BIAS, T_O, T_MLP_NORM, T_GATE_UP, T_DOWN = range(7)
T_EMBED, T_FINAL_NORM, T_LM_HEAD, T_PROMPT = 0xFFFF0001, 0xFFFF0002, 0xFFFF0003, 0xFFFF1000


def rbf(x: torch.Tensor) -> torch.Tensor:
    """Round fp32 through bf16 (the rounding point of a bf16 tensor op)."""
    return x.to(BF16).float()


def hash_tensor(shape, seed, tensor_id, scale, offset=0.0) -> torch.Tensor:
    n = int(np.prod(shape))
    bits = H.hash_bf16_bits(n, seed, tensor_id, scale, offset)
    return torch.from_numpy(bits.view(np.int16).copy()).view(BF16).reshape(shape)


def prompt(seed: int, request_id: int, length: int, vocab: int) -> torch.Tensor:
    return torch.from_numpy(H.hash_tokens(length, seed, T_PROMPT + request_id, vocab))


# ------------------------------------------------------------ kernel refs --

def rmsnorm_ref(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    var = xf.pow(2).mean(-1, keepdim=True)
    y = rbf(xf * torch.rsqrt(var + eps))
    return (w.float() * y).to(BF16)


_ACC = {"splits": 0}


class accumulation_order:
    """Context manager: linear layers sum K in `splits` fp32 partial products added in
    REVERSED order (a bf16-faithful variant that differs from the default single pass
    only in fp32 summation order -- the yardstick for the logits tolerance)."""

    def __init__(self, splits: int):
        self.splits = splits

    def __enter__(self):
        self.prev, _ACC["splits"] = _ACC["splits"], self.splits

    def __exit__(self, *exc):
        _ACC["splits"] = self.prev


def linear_acc(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """fp32 accumulator of x[T,K] . w[N,K]^T."""
    s = _ACC["splits"]
    if s <= 1:
        return x.float() @ w.float().t()
    K = x.shape[1]
    step = -(-K // s)
    parts = [x[:, k:k + step].float() @ w[:, k:k + step].float().t() for k in range(0, K, step)]
    acc = parts[-1]
    for p in reversed(parts[:-1]):
        acc = acc + p
    return acc


def swiglu_ref(acc_gate: torch.Tensor, acc_up: torch.Tensor) -> torch.Tensor:
    g, u = rbf(acc_gate), rbf(acc_up)
    return (rbf(torch.nn.functional.silu(g)) * u).to(BF16)


def deinterleave_gate_up(w_gu: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """[2 ffn, d] in 64-row blocks [gate|up] -> (W_gate [ffn, d], W_up [ffn, d])."""
    two_ffn, d = w_gu.shape
    blocks = w_gu.reshape(two_ffn // 128, 2, 64, d)
    return blocks[:, 0].reshape(-1, d), blocks[:, 1].reshape(-1, d)


def rope_table_ref(theta: float, hd: int, max_pos: int) -> torch.Tensor:
    inv_freq = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    ang = torch.arange(max_pos, dtype=torch.int64).float()[:, None] * inv_freq[None, :]
    return torch.cat([ang.cos(), ang.sin()], dim=1).to(BF16)


def rope_ref(x: torch.Tensor, pos: torch.Tensor, table: torch.Tensor) -> torch.Tensor:
    """x: [T, H, hd] bf16; neox rotate_half with per-op bf16 rounding."""
    hd = x.shape[-1]
    half = hd // 2
    cs = table[pos.long()].float()
    cos = cs[:, None, :half]
    sin = cs[:, None, half:]
    x1, x2 = x[..., :half].float(), x[..., half:].float()
    o1 = rbf(rbf(x1 * cos) + rbf(-x2 * sin))
    o2 = rbf(rbf(x2 * cos) + rbf(x1 * sin))
    return torch.cat([o1, o2], dim=-1).to(BF16)


def attention_ref(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal_offset: int | None) -> torch.Tensor:
    """q [Tq, Hq, hd], k/v [Tk, Hkv, hd] (bf16).  causal_offset: query i sees keys <= i + offset
    (None = all keys).  fp32 scores, softmax and P.V; output bf16 [Tq, Hq*hd]."""
    Tq, Hq, hd = q.shape
    Tk, Hkv, _ = k.shape
    G = Hq // Hkv
    qf = q.float().permute(1, 0, 2)                              # [Hq, Tq, hd]
    kf = k.float().permute(1, 0, 2).repeat_interleave(G, dim=0)  # [Hq, Tk, hd]
    vf = v.float().permute(1, 0, 2).repeat_interleave(G, dim=0)
    s = (qf @ kf.transpose(1, 2)) * (1.0 / math.sqrt(hd))
    if causal_offset is not None:
        qi = torch.arange(Tq)[:, None]
        kj = torch.arange(Tk)[None, :]
        s = s.masked_fill(kj > qi + causal_offset, float("-inf"))
    p = torch.softmax(s, dim=-1)
    o = p @ vf                                                    # [Hq, Tq, hd]
    return o.permute(1, 0, 2).reshape(Tq, Hq * hd).to(BF16)


# ------------------------------------------------------------ full model --

@dataclass
class OracleSpec:
    num_layers: int
    d: int
    Hq: int
    Hkv: int
    hd: int
    ffn: int
    vocab: int
    rope_theta: float
    eps: float
    qkv_bias: bool = False
    weight_scale: float = 0.02 * math.sqrt(3.0)
    embed_scale: float = 0.02 * math.sqrt(3.0)
    norm_jitter: float = 0.05
    bias_scale: float = 0.02
    peaked: bool = False
    lm_alpha: float = 4.0
    peaked_embed_scale: float = 8.0

    @classmethod
    def from_spec(cls, spec) -> "OracleSpec":
        return cls(**{f: getattr(spec, f) for f in cls.__dataclass_fields__})


@dataclass
class LayerW:
    attn_norm: torch.Tensor
    w_q: torch.Tensor
    w_k: torch.Tensor
    w_v: torch.Tensor
    b_q: torch.Tensor | None
    b_k: torch.Tensor | None
    b_v: torch.Tensor | None
    w_o: torch.Tensor
    mlp_norm: torch.Tensor
    w_gate: torch.Tensor
    w_up: torch.Tensor
    w_down: torch.Tensor


def make_layer(spec: OracleSpec, layer: int, seed: int, mk=None) -> LayerW:
    """Layer weights from the counter hash; `mk(shape, seed, tensor_id, scale, offset)`
    builds one tensor (default: the numpy generator)."""
    hash_tensor = mk or globals()["hash_tensor"]
    tid = lambda k: (layer << 4) | k  # noqa: E731
    s, d = spec.weight_scale, spec.d
    qkv_dim = (spec.Hq + 2 * spec.Hkv) * spec.hd
    w_qkv = hash_tensor((qkv_dim, d), seed, tid(T_QKV), s)
    q_rows, kv_rows = spec.Hq * spec.hd, spec.Hkv * spec.hd
    b = hash_tensor((qkv_dim,), seed, tid(T_QKV_BIAS), spec.bias_scale) if spec.qkv_bias else None
    gate, up = deinterleave_gate_up(hash_tensor((2 * spec.ffn, d), seed, tid(T_GATE_UP), s))
    return LayerW(
        attn_norm=hash_tensor((d,), seed, tid(T_ATTN_NORM), spec.norm_jitter, 1.0),
        w_q=w_qkv[:q_rows], w_k=w_qkv[q_rows:q_rows + kv_rows], w_v=w_qkv[q_rows + kv_rows:],
        b_q=None if b is None else b[:q_rows],
        b_k=None if b is None else b[q_rows:q_rows + kv_rows],
        b_v=None if b is None else b[q_rows + kv_rows:],
        w_o=hash_tensor((d, spec.Hq * spec.hd), seed, tid(T_O), s),
        mlp_norm=hash_tensor((d,), seed, tid(T_MLP_NORM), spec.norm_jitter, 1.0),
        w_gate=gate, w_up=up,
        w_down=hash_tensor((d, spec.ffn), seed, tid(T_DOWN), s),
    )


def make_embed(spec: OracleSpec, seed: int, mk=None) -> torch.Tensor:
    hash_tensor = mk or globals()["hash_tensor"]
    scale = spec.peaked_embed_scale if spec.peaked else spec.embed_scale
    return hash_tensor((spec.vocab, spec.d), seed, T_EMBED, scale)


def make_head(spec: OracleSpec, seed: int, mk=None) -> tuple[torch.Tensor, torch.Tensor]:
    hash_tensor = mk or globals()["hash_tensor"]
    final_norm = hash_tensor((spec.d,), seed, T_FINAL_NORM, spec.norm_jitter, 1.0)
    if spec.peaked:
        e = make_embed(spec, seed, mk)
        lm = (torch.roll(e, shifts=-1, dims=0).float() * spec.lm_alpha).to(BF16)
    else:
        lm = hash_tensor((spec.vocab, spec.d), seed, T_LM_HEAD, spec.weight_scale)
    return final_norm, lm


def _proj(x, w, b):
    acc = linear_acc(x, w)
    if b is not None:
        acc = acc + b.float()
    return acc.to(BF16)


def layer_forward(spec: OracleSpec, W: LayerW, h: torch.Tensor, pos: torch.Tensor, table,
                  cache: list[tuple[torch.Tensor, torch.Tensor]], seg: list[int]) -> torch.Tensor:
    """One decoder layer over a varlen batch.  h [T, d] bf16 rows grouped per request by
    `seg` (token counts); `cache[r]` = (k, v) of request r before this call, extended in place."""
    a = rmsnorm_ref(h, W.attn_norm, spec.eps)
    T = h.shape[0]
    q = _proj(a, W.w_q, W.b_q).reshape(T, spec.Hq, spec.hd)
    k = _proj(a, W.w_k, W.b_k).reshape(T, spec.Hkv, spec.hd)
    v = _proj(a, W.w_v, W.b_v).reshape(T, spec.Hkv, spec.hd)
    q, k = rope_ref(q, pos, table), rope_ref(k, pos, table)
    outs = []
    off = 0
    for r, n in enumerate(seg):
        kc, vc = cache[r]
        kc = torch.cat([kc, k[off:off + n]], 0)
        vc = torch.cat([vc, v[off:off + n]], 0)
        cache[r] = (kc, vc)
        past = kc.shape[0] - n
        outs.append(attention_ref(q[off:off + n], kc, vc, causal_offset=past))
        off += n
    o = torch.cat(outs, 0)
    h = (rbf(linear_acc(o, W.w_o)) + h.float()).to(BF16)
    a = rmsnorm_ref(h, W.mlp_norm, spec.eps)
    m = swiglu_ref(linear_acc(a, W.w_gate), linear_acc(a, W.w_up))
    return (rbf(linear_acc(m, W.w_down)) + h.float()).to(BF16)


@dataclass
class OracleModel:
    """CPU decoder for a layer range [lo, hi) (whole model by default)."""

    spec: OracleSpec
    seed: int = 0
    lo: int = 0
    hi: int | None = None
    max_pos: int = 4096
    layers: list[LayerW] = field(default_factory=list)

    def __post_init__(self):
        if self.hi is None:
            self.hi = self.spec.num_layers
        self.layers = [make_layer(self.spec, l, self.seed) for l in range(self.lo, self.hi)]
        self.embed = make_embed(self.spec, self.seed)
        self.final_norm, self.lm_head = make_head(self.spec, self.seed)
        self.table = rope_table_ref(self.spec.rope_theta, self.spec.hd, self.max_pos)

    def new_cache(self, n_req: int):
        e = torch.empty(0, self.spec.Hkv, self.spec.hd, dtype=BF16)
        return [[(e, e) for _ in range(n_req)] for _ in self.layers]

    def forward(self, tokens: list[torch.Tensor], positions: list[torch.Tensor], caches) -> torch.Tensor:
        """Embed + all layers + final norm + fp32 logits at each request's last row."""
        ids = torch.cat(tokens)
        pos = torch.cat(positions)
        seg = [t.numel() for t in tokens]
        h = self.embed[ids]
        for i, W in enumerate(self.layers):
            h = layer_forward(self.spec, W, h, pos, self.table, caches[i], seg)
        last = torch.tensor(np.cumsum(seg) - 1)
        hn = rmsnorm_ref(h[last], self.final_norm, self.spec.eps)
        return linear_acc(hn, self.lm_head)

    def greedy(self, prompts: list[torch.Tensor], n_new: int):
        """Greedy decode every request (rows are independent; batching does not change values).
        Returns (tokens [R, n_new] int64, logits list per step [R, V] fp32)."""
        R = len(prompts)
        caches = self.new_cache(R)
        logits = self.forward(prompts, [torch.arange(p.numel()) for p in prompts], caches)
        out, all_logits = [logits.argmax(-1)], [logits]
        for step in range(1, n_new):
            toks = [out[-1][r:r + 1] for r in range(R)]
            pos = [torch.tensor([prompts[r].numel() + step - 1]) for r in range(R)]
            logits = self.forward(toks, pos, caches)
            out.append(logits.argmax(-1))
            all_logits.append(logits)
        return torch.stack(out, 1), all_logits

    def teacher_forced(self, prompt_ids: torch.Tensor, generated: torch.Tensor) -> torch.Tensor:
        """fp32 logits predicting generated[i] given prompt + generated[:i] (one causal pass)."""
        seq = torch.cat([prompt_ids, generated[:-1]])
        caches = self.new_cache(1)
        ids, pos = seq, torch.arange(seq.numel())
        h = self.embed[ids]
        for i, W in enumerate(self.layers):
            h = layer_forward(self.spec, W, h, pos, self.table, caches[i], [seq.numel()])
        rows = torch.arange(prompt_ids.numel() - 1, seq.numel())
        hn = rmsnorm_ref(h[rows], self.final_norm, self.spec.eps)
        return linear_acc(hn, self.lm_head)


# ------------------------------------------------------ layer-streamed model --

def torch_hash_maker(device="cpu"):
    """Tensor factory for make_layer & co. on torch (host threads or a GPU's elementwise
    ops): bit-identical to hash_tensor, the result always on the host."""
    def mk(shape, seed, tensor_id, scale, offset=0.0):
        return H.hash_bf16_torch(tuple(shape), seed, tensor_id, scale, offset, device=device).cpu()
    return mk


def stream_forward(spec: OracleSpec, seed: int, seqs: list[torch.Tensor], rows: list[torch.Tensor],
                   mk=None, lo: int = 0, hi: int | None = None, max_pos: int = 4096):
    """Whole-model causal forward of independent sequences, ONE LAYER RESIDENT AT A TIME
    (a 32-layer Llama-3-8B or an 80-layer Qwen2-72B slice never sits in host memory at
    once).  Returns (hn [sum rows, d] bf16 after the final norm, fp32 logits) at the
    positions `rows[i]` of sequence i -- e.g. the rows predicting each generated token."""
    hi = spec.num_layers if hi is None else hi
    table = rope_table_ref(spec.rope_theta, spec.hd, max_pos)
    ids = torch.cat(seqs)
    pos = torch.cat([torch.arange(s.numel()) for s in seqs])
    seg = [s.numel() for s in seqs]
    h = make_embed(spec, seed, mk)[ids]
    e = torch.empty(0, spec.Hkv, spec.hd, dtype=BF16)
    for l in range(lo, hi):
        W = make_layer(spec, l, seed, mk)
        h = layer_forward(spec, W, h, pos, table, [(e, e) for _ in seqs], seg)
        del W
    off = np.concatenate([[0], np.cumsum(seg)[:-1]])
    sel = torch.cat([torch.as_tensor(r, dtype=torch.int64) + int(o) for r, o in zip(rows, off)])
    final_norm, lm_head = make_head(spec, seed, mk)
    hn = rmsnorm_ref(h[sel], final_norm, spec.eps)
    return hn, linear_acc(hn, lm_head)
