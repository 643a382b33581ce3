"""Helper for bit-identity tests across GEMM policies (run in a subprocess, since the
policies are read from the environment once per process):

    PL_CSK=0 python tests/_stage_steps.py out.pt

One 2-layer Llama-3-shape stage: a prefill forward (R requests, T tokens: decode-
orientation GEMMs with split-K, QKV+RoPE+KV-append and residual+norm fusions), then
three decode forwards over the KV it wrote.  Saves every step's hidden state and ids.
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_05043_b200 import LLAMA3_8B  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor, build_meta  # noqa: E402
from paper_2507_05043_b200.spec import prompt_tokens  # noqa: E402


def main(out_path, T=64, R=4):
    spec = LLAMA3_8B.with_(num_layers=2)
    exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, torch.device("cuda", 0), seed=0,
                        pack_weights=True, max_tokens=max(T, 16), max_reqs=R, max_ctx=512, num_blocks=R * 8,
                        n_slots=1)
    lens = [T // R] * R
    lens[-1] += T - sum(lens)
    rows = np.arange(R * exe.max_blocks, dtype=np.int32).reshape(R, -1)
    cu = np.concatenate([[0], np.cumsum(lens)])
    pos = np.concatenate([np.arange(n) for n in lens])
    req_of = np.repeat(np.arange(R), lens)
    slots = rows[req_of, pos // 64] * 64 + pos % 64
    meta = build_meta(T, R, exe.max_blocks, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
    ids = np.concatenate([prompt_tokens(0, i, n, spec.vocab) for i, n in enumerate(lens)])
    exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
    exe.ids_dev[:T].copy_(torch.from_numpy(ids))
    torch.cuda.synchronize()
    exe.forward(0, T, R, False, max(lens), max(lens))
    exe.stream.synchronize()
    outs = [exe.hidden[0][:T].clone().cpu(), exe.out_ids[0][:R].clone().cpu()]
    ctx = np.array(lens)
    last = torch.zeros(R, dtype=torch.int64, device="cuda:0")
    for _ in range(3):  # decode steps over the KV pages the prefill (and earlier steps) wrote
        last.copy_(exe.out_ids[0][:R])
        p = ctx.copy()
        sl = rows[np.arange(R), p // 64] * 64 + p % 64
        ctx = ctx + 1
        meta = build_meta(R, R, exe.max_blocks, p, sl, np.arange(R), np.arange(R + 1), ctx, np.arange(R), rows)
        exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
        torch.cuda.synchronize()
        exe.forward(0, R, R, True, 1, int(ctx.max()), last_token=last)
        exe.stream.synchronize()
        outs += [exe.hidden[0][:R].clone().cpu(), exe.out_ids[0][:R].clone().cpu()]
    torch.save(outs, out_path)


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:]))
