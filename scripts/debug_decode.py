"""Debug: one decode step through pl_stage_forward vs the same layer math composed
from individually tested ops.* kernels, layer by layer (tiny model)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_05043_b200 import TINY, ops  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor, build_meta  # noqa: E402
from paper_2507_05043_b200.spec import prompt_tokens  # noqa: E402


def main(n_layers):
    spec = TINY.with_(num_layers=n_layers)
    lens = [100, 37, 64]
    R, T = len(lens), sum(lens)
    exe = StageExecutor(spec, 0, (0, n_layers), True, True, torch.device("cuda", 0), seed=0,
                        max_tokens=T, max_reqs=R, max_ctx=256, num_blocks=12, n_slots=1)
    mb_ = exe.max_blocks
    rows = np.arange(R * mb_, dtype=np.int32).reshape(R, -1)
    cu = np.concatenate([[0], np.cumsum(lens)])
    pos = np.concatenate([np.arange(n) for n in lens])
    req_of = np.repeat(np.arange(R), lens)
    slots = rows[req_of, pos // 64] * 64 + pos % 64
    ids = np.concatenate([prompt_tokens(0, i, n, spec.vocab) for i, n in enumerate(lens)])
    meta = build_meta(T, R, mb_, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
    exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
    exe.ids_dev[:T].copy_(torch.from_numpy(ids))
    torch.cuda.synchronize()
    exe.forward(0, T, R, False, max(lens), max(lens))
    torch.cuda.synchronize()
    kv_after_prefill = [(L["k_cache"].clone(), L["v_cache"].clone()) for L in exe.layers]
    nxt = exe.out_ids[0][:R].clone()

    # decode step via the stage
    p = np.array(lens)
    dslots = rows[np.arange(R), p // 64] * 64 + p % 64
    meta = build_meta(R, R, mb_, p, dslots, np.arange(R), np.arange(R + 1), p + 1, np.arange(R), rows)
    exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
    torch.cuda.synchronize()
    exe.forward(0, R, R, True, 1, int(p.max()) + 1, last_token=nxt)
    torch.cuda.synchronize()
    h_stage = exe.hidden[0][:R].float().clone()

    # same step composed from ops (on a copy of the post-prefill caches)
    dev = exe.device
    h = exe.embed[nxt]
    pos_d = torch.tensor(p, dtype=torch.int32, device=dev)
    slot_d = torch.tensor(dslots, dtype=torch.int32, device=dev)
    bt = torch.tensor(rows, dtype=torch.int32, device=dev)
    ctx = torch.tensor(p + 1, dtype=torch.int32, device=dev)
    for l, L in enumerate(exe.layers):
        kc, vc = (x.clone() for x in kv_after_prefill[l])
        a = ops.rmsnorm(h, L["attn_norm"], spec.eps)
        qkv = ops.gemm(a, L["w_qkv"])
        ops.rope_kv_write(qkv, pos_d, slot_d, exe.cos_sin, kc, vc, spec.Hq, spec.Hkv, spec.hd)
        o = ops.attn_decode(qkv, kc, vc, bt, ctx, int(p.max()) + 1, spec.Hq, spec.Hkv, spec.hd)
        h = h.clone()
        ops.gemm(o, L["w_o"], ops.EPI_RESIDUAL, residual=h, out=h)
        a = ops.rmsnorm(h, L["mlp_norm"], spec.eps)
        m = ops.gemm(a, L["w_gate_up"], ops.EPI_SWIGLU)
        ops.gemm(m, L["w_down"], ops.EPI_RESIDUAL, residual=h, out=h)
        kdiff = (kc.float() - L["k_cache"].float()).abs().max().item()
        print(f"layer {l}: k-cache diff {kdiff:.4g}")
    torch.cuda.synchronize()
    print("max |h_stage - h_ops| =", (h_stage - h.float()).abs().max().item(),
          " |h| max", h.float().abs().max().item())


if __name__ == "__main__":
    for n in (1, 4):
        main(n)
