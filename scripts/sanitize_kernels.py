"""One small invocation of every libb200link kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_kernels.py

Covers: tcgen05 GEMMs (decode SWAP split-K with the residual+norm reduce, cluster
split-K over DSMEM with RoPE/KV append, packed bulk-copy weights, argmax), the
prefill GEMM on CTA pairs (cta_group::2), decode attention (TMA pages, split merge),
prefill attention, RMSNorm / RoPE / embed / token scatter, and one decode forward of
a 2-layer stage through the persistent chain kernel (PL_CHAIN=1 set below).
"""

import os
import sys
from pathlib import Path

os.environ.setdefault("PL_CHAIN", "1")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B, TINY, ops  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402
from paper_2507_05043_b200.profiler import time_forward  # noqa: E402
from paper_2507_05043_b200.spec import prompt_tokens  # noqa: E402

d = torch.device("cuda", 0)
B = torch.bfloat16
g = torch.Generator().manual_seed(0)
r = lambda *s: (torch.randn(*s, generator=g) * 0.05).to(B).to(d)  # noqa: E731

# GEMMs: decode split-K + residual, plain, bias; prefill single CTA and CTA pair; argmax
x, w = r(24, 1024), r(768, 1024)
h = r(24, 768)
ops.gemm(x, w)
ops.gemm(x, w, ops.EPI_RESIDUAL, residual=h, out=h)
ops.gemm(r(600, 512), r(512, 512))
ops.gemm(r(300, 256), r(256, 256), ops.EPI_BIAS, bias=r(256))
ops.gemm_packed(x, ops.pack_weight(r(1024, 1024)))
ops.lmhead_argmax(r(5, 256), r(2048, 256))
ops.rmsnorm(r(9, 256), r(256), 1e-5)
# attention: decode (split: > 1024-token contexts) and prefill
Hq, Hkv, hd = 4, 2, 128
ctx = torch.tensor([1100, 70], dtype=torch.int32)
nb = 24
bt = torch.arange(2 * 18, dtype=torch.int32).reshape(2, 18) % nb
ops.attn_decode(r(2, Hq * hd), r(nb, Hkv, 64, hd), r(nb, Hkv, 64, hd), bt.to(d), ctx.to(d), 1100, Hq, Hkv, hd)
ops.attn_prefill(r(200, (Hq + 2 * Hkv) * hd), torch.tensor([0, 77, 200], dtype=torch.int32, device=d), 123,
                 Hq, Hkv, hd)
torch.cuda.synchronize()

# whole-stage forwards: tiny (prefill + decode through the chain kernel) and a 2-layer
# Llama-3-8B-shape stage (cluster split-K QKV + RoPE/KV append at T = 32, CTA pairs at 512)
for spec, T in ((TINY, 8), (LLAMA3_8B.with_(num_layers=2), 32)):
    exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, d, max_tokens=512, max_reqs=T,
                        max_ctx=200, num_blocks=T * 4 + 8, n_slots=1)
    time_forward(exe, T, True, ctx=150, reps=1)
    time_forward(exe, 512, False, reps=1)
    ids, hn = exe.greedy([prompt_tokens(0, i, 40 + i, spec.vocab) for i in range(3)], 3)
    exe.close()
torch.cuda.synchronize()
print("sanitize workload done")
