"""Full-depth parity of the benched models at STANDARD init.

The bench times the whole 32-layer Llama-3-8B-shape model with std-0.02 weights;
accumulation-order differences compound over depth, so this checks that model
itself (and a 10-layer Qwen2-72B-shape slice with qkv bias, one S=8 stage's
depth) end to end on the GPU against the layer-streamed CPU oracle:

* GPU: one stage holding the whole model (embed .. lm_head) runs a prefill of 4
  hash prompts (64..112 tokens -> a 352-token prefill micro-batch) and 3 decode
  micro-batches fed its own greedy ids (StageExecutor.greedy).
* Oracle: oracle/decoder.stream_forward teacher-forced on the GPU's ids (one
  layer resident at a time, weights from the torch restatement of the hash
  initialiser -- bit-identical to the GPU fill, tests/test_oracle_hash.py).
* logits: both sides' final-normed rows times the same lm_head in fp32 on the
  host; max |dlogit| <= tol, where tol = 4x the drift between two CPU oracles
  that differ only in fp32 summation order, through the same model and
  workload (tests/golden/logit_tolerance.json, oracle/calibrate_tolerance.py).
* greedy ids: every GPU id lies inside the oracle's tie band (its oracle logit
  is within tol of the row max); exact matches are reported (two CPU oracles that
  differ only in summation order already disagree on 4/32 (L3) and 8/32 (Q2)
  argmaxes of this workload at standard init -- logit_tolerance.json -- so exact
  identity is asserted only under the margin-engineered init, below).
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import decoder as OD

pytestmark = pytest.mark.gpu

TOL = json.loads((Path(__file__).resolve().parent / "golden" / "logit_tolerance.json").read_text())


def full_model_check(spec, name, R=4, steps=4, seed=0):
    from paper_2507_05043_b200.executor import StageExecutor
    from paper_2507_05043_b200.spec import prompt_tokens

    lens = [64 + 16 * r for r in range(R)]
    prompts = [prompt_tokens(seed, r, n, spec.vocab) for r, n in enumerate(lens)]
    blocks = sum(-(-(n + steps) // 64) for n in lens)
    exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, torch.device("cuda", 0), seed=seed,
                        max_tokens=sum(lens), max_reqs=R, max_ctx=max(lens) + steps, num_blocks=blocks,
                        n_slots=1)
    ids, hn = exe.greedy(prompts, steps)
    exe.close()
    del exe
    torch.cuda.empty_cache()

    o = OD.OracleSpec.from_spec(spec)
    mk = OD.torch_hash_maker("cuda")
    seqs = [torch.cat([torch.from_numpy(p), torch.from_numpy(ids[r, :-1])]) for r, p in enumerate(prompts)]
    rows = [torch.arange(n - 1, n - 1 + steps) for n in lens]
    hn_ref, ref = OD.stream_forward(o, seed, seqs, rows, mk=mk, max_pos=max(lens) + steps + 1)
    _, lm = OD.make_head(o, seed, mk)
    got = OD.linear_acc(hn.permute(1, 0, 2).reshape(R * steps, -1), lm)
    err = (got - ref).abs().max().item()
    tol = TOL[name]["tol"]
    chosen = ref.gather(1, torch.from_numpy(ids.reshape(-1)).long()[:, None]).squeeze(1)
    gap = (ref.max(-1).values - chosen).max().item()
    exact = int((ref.argmax(-1).numpy() == ids.reshape(-1)).sum())
    print(f"{name}: max|dlogit| {err:.5f} (tol {tol:.5f}, logit std {ref.std():.3f}); tie gap {gap:.5f}; "
          f"exact {exact}/{ids.size}")
    return err, tol, gap, exact, ids.size


def test_llama3_8b_full_depth_standard_init():
    from paper_2507_05043_b200 import LLAMA3_8B

    err, tol, gap, exact, n = full_model_check(LLAMA3_8B, "l3-32")
    assert err <= tol, f"max |dlogit| {err:.5f} > tol {tol:.5f}"
    assert gap <= tol, f"a GPU token sits {gap:.5f} below the oracle max (band {tol:.5f})"
    assert exact >= n // 2


def test_qwen2_72b_ten_layer_slice_standard_init():
    from paper_2507_05043_b200 import QWEN2_72B

    err, tol, gap, exact, n = full_model_check(QWEN2_72B.with_(num_layers=10), "q2-10")
    assert err <= tol, f"max |dlogit| {err:.5f} > tol {tol:.5f}"
    assert gap <= tol, f"a GPU token sits {gap:.5f} below the oracle max (band {tol:.5f})"
    assert exact >= n // 2


@pytest.mark.parametrize("name", ["l3-32", "q2-10"])
def test_full_depth_peaked_greedy_identical(name):
    """Margin-engineered init (embed U(+-8), lm_head[v] = 4 embed[v+1]):
    the benched depths produce greedy ids IDENTICAL to the oracle's -- the oracle's
    teacher-forced argmax equals the GPU's id at every step, i.e. the oracle's own
    greedy sequence is the GPU's."""
    from paper_2507_05043_b200 import LLAMA3_8B, QWEN2_72B

    spec = (LLAMA3_8B if name == "l3-32" else QWEN2_72B.with_(num_layers=10)).with_(peaked=True)
    err, tol, gap, exact, n = full_model_check(spec, name)
    assert exact == n, f"{n - exact} of {n} greedy ids differ from the oracle"
