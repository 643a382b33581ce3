"""ORACLE (bench CPU-baseline leg only): time the CPU decoder on the host cores.

The reference has no CPU forward (its compute is a latency table,
pipelink/engine.py:384), so the CPU baseline is this repo's oracle decoder
(oracle/decoder.py) run with all host threads.  A full Llama-3-8B-shape
serving run would take tens of minutes on CPU, so the estimate is built from
bounded samples of the SAME workload and extrapolated:

  * decode: one decode step of B requests at the run's MEAN context
    (P + (n_out - 1) / 2: decode attention is linear in the context, so the mean
    step is the average step) through `layers_sampled` decoder layers, plus
    embed + final norm + lm_head;
  * prefill: one whole prompt of P tokens through the sampled layers (the causal
    attention's quadratic term is timed, not extrapolated); prompts longer than
    `prefill_cap` are sampled at the cap and scaled linearly (said in `sample`).

  t_decode_step = t_head + L/ls * t_layers(decode at the mean context)
  t_prefill     = B * (L/ls * t_layers(prefill of one prompt) + t_head')
  output tok/s  = B * n_out / (t_prefill + (n_out - 1) * t_decode_step)

Weights for the TIMING sample are drawn with torch's RNG (values do not change
CPU time); the oracle code path timed is the one the parity tests use.
"""

from __future__ import annotations

import os
import time

import torch

from . import decoder as OD

BF16 = torch.bfloat16


def _rand_layer(spec: OD.OracleSpec, g: torch.Generator) -> OD.LayerW:
    s = spec.weight_scale
    f = lambda *shape: (torch.rand(*shape, generator=g) * 2 - 1).mul_(s).to(BF16).float()  # noqa: E731
    qd, kd = spec.Hq * spec.hd, spec.Hkv * spec.hd
    ones = torch.ones(spec.d)
    b = (lambda n: f(n)) if spec.qkv_bias else (lambda n: None)
    return OD.LayerW(attn_norm=ones, w_q=f(qd, spec.d), w_k=f(kd, spec.d), w_v=f(kd, spec.d),
                     b_q=b(qd), b_k=b(kd), b_v=b(kd), w_o=f(spec.d, qd), mlp_norm=ones,
                     w_gate=f(spec.ffn, spec.d), w_up=f(spec.ffn, spec.d), w_down=f(spec.d, spec.ffn))


def estimate(spec, batch: int, prompt_len: int, n_out: int, layers_sampled: int = 2,
             prefill_cap: int = 1024, threads: int | None = None, reps: int = 2) -> dict:
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    o = OD.OracleSpec.from_spec(spec)
    g = torch.Generator().manual_seed(0)
    ls = min(layers_sampled, o.num_layers)
    layers = [_rand_layer(o, g) for _ in range(ls)]
    emb = (torch.rand(o.vocab, o.d, generator=g) * 0.07 - 0.035).to(BF16)
    lm = (torch.rand(o.vocab, o.d, generator=g) * 0.07 - 0.035).to(BF16).float()
    fnorm = torch.ones(o.d)
    table = OD.rope_table_ref(o.rope_theta, o.hd, prompt_len + n_out + 1)

    def head(h):
        hn = OD.rmsnorm_ref(h, fnorm, o.eps)
        return OD.linear_acc(hn, lm).argmax(-1)

    # decode step: B requests, one token each, at the run's mean context
    ctx = prompt_len + (n_out - 1) // 2
    kv = [[((torch.randn(ctx, o.Hkv, o.hd, generator=g) * 0.5).to(BF16),
            (torch.randn(ctx, o.Hkv, o.hd, generator=g) * 0.5).to(BF16))
           for _ in range(batch)] for _ in range(ls)]
    ids = torch.randint(0, o.vocab, (batch,), generator=g)
    pos = torch.full((batch,), ctx, dtype=torch.int64)

    def decode_once():
        caches = [[c for c in layer] for layer in kv]   # fresh lists: layer_forward appends
        t0 = time.perf_counter()
        h = emb[ids]
        for i, W in enumerate(layers):
            h = OD.layer_forward(o, W, h, pos, table, caches[i], [1] * batch)
        t1 = time.perf_counter()
        head(h)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    def prefill_once():
        n = min(prefill_cap, prompt_len)
        tok = torch.randint(0, o.vocab, (n,), generator=g)
        e = torch.empty(0, o.Hkv, o.hd, dtype=BF16)
        caches = [[(e, e)] for _ in range(ls)]
        t0 = time.perf_counter()
        h = emb[tok]
        for i, W in enumerate(layers):
            h = OD.layer_forward(o, W, h, torch.arange(n), table, caches[i], [n])
        t1 = time.perf_counter()
        head(h[-1:])
        t2 = time.perf_counter()
        return (t1 - t0) * prompt_len / n, t2 - t1  # one whole prompt

    decode_once()  # warm
    d = min((decode_once() for _ in range(reps)), key=lambda x: x[0] + x[1])
    p = min((prefill_once() for _ in range(reps)), key=lambda x: x[0])
    scale = o.num_layers / ls
    t_step = d[0] * scale + d[1]
    t_prefill = batch * (p[0] * scale + p[1])
    total_tokens = batch * n_out
    t_run = t_prefill + (n_out - 1) * t_step
    return {
        "tok_s": total_tokens / t_run,
        "decode_tok_s": batch / t_step,
        "t_decode_step_s": t_step,
        "t_prefill_s": t_prefill,
        "threads": threads,
        "sample": (f"oracle CPU decoder: 1 decode step of B={batch} at the mean ctx {ctx} and one "
                   f"{min(prefill_cap, prompt_len)}-token prefill"
                   f"{'' if prompt_len <= prefill_cap else ' (scaled linearly to ' + str(prompt_len) + ')'}"
                   f" through {ls}/{o.num_layers} layers + lm_head, extrapolated to the full "
                   f"{batch}x{prompt_len}/{n_out} run"),
    }
