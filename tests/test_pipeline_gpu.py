"""End-to-end parity of the B200 pipeline against the CPU oracle.

* schedule: the run's RunResult equals pipelink.PipelineEngine.run for the same
  profiles (bit-exact, decisions are virtual-clock);
* greedy token ids: identical to the oracle under the margin-engineered
  ("peaked") init, on config 1 (tiny, S=2) and on a truncated Llama-3-8B-shape
  model; under the standard init every GPU token lies inside the oracle's tie
  band (teacher forced) and >= 90% match exactly;
* logits: the GPU stack's fp32 logits are within |dlogit| <= tol of the oracle's
  (bf16 rounding points identical, fp32 summation order differs); tol = 4x the
  drift between two CPU oracles that differ only in summation order
  (tests/golden/logit_tolerance.json, oracle/calibrate_tolerance.py).
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

import pipelink
from oracle import decoder as OD

from paper_2507_05043_b200 import LLAMA3_8B, TINY, deploy, ops
from paper_2507_05043_b200.engine import B200PipelineEngine
from paper_2507_05043_b200.executor import StageExecutor, build_meta
from paper_2507_05043_b200.spec import prompt_tokens
from test_driver_parity import result_key

pytestmark = pytest.mark.gpu

_TOL = json.loads((Path(__file__).resolve().parent / "golden" / "logit_tolerance.json").read_text())


def tol_of(spec) -> float:
    """Calibrated logits tolerance of a test model (see the module docstring)."""
    key = "tiny" if spec.d == 256 else "tiny-d1024" if spec.d == 1024 else None
    return _TOL[key]["tol"]


def synth_profiles(plan, per_token=1e-6, overhead=2e-5):
    return [pipelink.synth_profile(hi - lo, per_token, overhead, stage_id=i)
            for i, (_, (lo, hi)) in enumerate(plan.stages)]


def config1(spec, S=2, n_req=8, in_len=128, out_len=32, mbt=1024, chunk=pipelink.DEFAULT_CHUNK_SIZE):
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    ctrl = pipelink.ControllerConfig(max_batched_tokens=mbt, max_batch_size=n_req)
    cfg = deploy.engine_config(plan, spec, ctrl, chunk_size=chunk)
    return cfg, cluster, plan, deploy.uniform_trace(n_req, in_len, out_len)


def run_gpu(spec, cfg, cluster, plan, trace, seed=0, native=True):
    profiles = synth_profiles(plan)
    eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec, seed=seed, native=native)
    res = eng.run(trace)
    ref = pipelink.PipelineEngine(cfg, cluster, profiles).run(trace)
    a, b = result_key(ref), result_key(res)
    for k in a:
        assert a[k] == b[k], f"schedule mismatch in {k}"
    assert res.all_finished
    eng.close()
    return res


def oracle_greedy(spec, trace, seed=0, lo=0, hi=None):
    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=seed, lo=lo, hi=hi, max_pos=2048)
    prompts = [torch.from_numpy(prompt_tokens(seed, r.id, r.input_len, spec.vocab)) for r in trace.requests]
    out_len = trace.requests[0].output_len
    toks, logits = model.greedy(prompts, out_len)
    return model, prompts, toks


@pytest.mark.parametrize("native", [True, False], ids=["native", "python"])
def test_config1_peaked_tokens_identical(native):
    """Native C++ runtime and the Python driver twin: same schedule, same tokens."""
    spec = TINY.with_(peaked=True)
    cfg, cluster, plan, trace = config1(spec)
    res = run_gpu(spec, cfg, cluster, plan, trace, native=native)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        got = res.b200.tokens[r.id]
        assert len(got) == r.output_len
        assert np.array_equal(got, want[i].numpy()), f"request {r.id}: {got[:8]} vs {want[i][:8]}"


def test_config1_standard_init_tie_band():
    spec = TINY
    cfg, cluster, plan, trace = config1(spec)
    res = run_gpu(spec, cfg, cluster, plan, trace)
    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=2048)
    exact = total = 0
    for r in trace.requests:
        gen = torch.from_numpy(res.b200.tokens[r.id])
        p = torch.from_numpy(prompt_tokens(0, r.id, r.input_len, spec.vocab))
        logits = model.teacher_forced(p, gen)          # [out_len, V]
        best = logits.max(-1).values
        chosen = logits.gather(1, gen[:, None]).squeeze(1)
        tol = tol_of(spec)
        gap = (best - chosen).max().item()
        assert (chosen >= best - tol).all(), f"request {r.id}: token {gap:.4f} below the max (band {tol:.4f})"
        exact += (logits.argmax(-1) == gen).sum().item()
        total += gen.numel()
    assert exact / total >= 0.9, f"only {exact}/{total} exact"


@pytest.mark.parametrize("spec_name,T", [("tiny", 64), ("l3-2", 64), ("l3-2", 300), ("l3-2", 600)])
def test_packed_weights_bit_identical(spec_name, T):
    """Pre-swizzled weight tiles (bulk copies) vs row-major weights (TMA boxes): the
    same tiles reach the tensor cores in the same order, so hidden states and token
    ids are bit-identical -- decode (SWAP) and prefill (T > 256) orientations, the latter
    on CTA pairs at T >= 512 (packed tiles as a 3-D TMA box)."""
    spec = TINY if spec_name == "tiny" else LLAMA3_8B.with_(num_layers=2)
    R = 4
    lens = [T // R] * R
    lens[-1] += T - sum(lens)
    outs = []
    for pack in (False, True):
        exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, torch.device("cuda", 0), seed=0,
                            pack_weights=pack, max_tokens=T, max_reqs=R, max_ctx=512, num_blocks=64,
                            n_slots=1)
        cu = np.concatenate([[0], np.cumsum(lens)])
        pos = np.concatenate([np.arange(n) for n in lens])
        rows = np.arange(R * exe.max_blocks, dtype=np.int32).reshape(R, -1)
        req_of = np.repeat(np.arange(R), lens)
        slots = rows[req_of, pos // 64] * 64 + pos % 64
        meta = build_meta(T, R, exe.max_blocks, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
        ids = np.concatenate([prompt_tokens(0, i, n, spec.vocab) for i, n in enumerate(lens)])
        exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
        exe.ids_dev[:T].copy_(torch.from_numpy(ids))
        torch.cuda.synchronize()
        exe.forward(0, T, R, False, max(lens), max(lens))
        exe.stream.synchronize()
        outs.append((exe.hidden[0][:T].clone().cpu(), exe.out_ids[0][:R].clone().cpu()))
        exe.close()
        del exe
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1], outs[1][1])


def test_stage_logits_within_tolerance():
    """Whole tiny model as one stage: GPU residual stream + GPU logits vs the oracle."""
    spec = TINY
    lens = [128, 77, 3]
    R, T = len(lens), sum(lens)
    exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, torch.device("cuda", 0), seed=0,
                        pack_weights=False,
                        max_tokens=T, max_reqs=R, max_ctx=256, num_blocks=16, n_slots=1)
    cu = np.concatenate([[0], np.cumsum(lens)])
    pos = np.concatenate([np.arange(n) for n in lens])
    rows = np.arange(R * exe.max_blocks, dtype=np.int32).reshape(R, -1)
    req_of = np.repeat(np.arange(R), lens)
    slots = rows[req_of, pos // 64] * 64 + pos % 64
    meta = build_meta(T, R, exe.max_blocks, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
    ids = np.concatenate([prompt_tokens(0, i, n, spec.vocab) for i, n in enumerate(lens)])
    exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
    exe.ids_dev[:T].copy_(torch.from_numpy(ids))
    torch.cuda.synchronize()
    exe.forward(0, T, R, False, max(lens), max(lens))
    exe.stream.synchronize()
    hidden = exe.hidden[0][:T].clone()
    last = torch.tensor(cu[1:] - 1, dtype=torch.int32, device=hidden.device)
    hn = ops.rmsnorm(hidden, exe.final_norm, spec.eps, row_idx=last)
    ids_gpu = exe.out_ids[0][:R].cpu()

    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=256)
    toks = [torch.from_numpy(ids[cu[i]:cu[i + 1]]) for i in range(R)]
    ref = model.forward(toks, [torch.arange(n) for n in lens], model.new_cache(R))
    # GPU logits from the GPU's final-normed rows in fp32 (the lm_head GEMM's bf16 store
    # epilogue would add a rounding the argmax path never sees)
    logits = OD.linear_acc(hn.cpu(), exe.lm_head.cpu())
    err = (logits - ref).abs().max().item()
    tol = tol_of(spec)
    assert err <= tol, f"max |dlogit| {err:.4f} (tol {tol:.4f})"
    top2 = ref.topk(2, -1).values
    clear = (top2[:, 0] - top2[:, 1]) > tol
    assert torch.equal(ids_gpu[clear], ref.argmax(-1)[clear])
    exe.close()


@pytest.mark.parametrize("pack", [False, True], ids=["rowmajor", "chain"])
@pytest.mark.parametrize("spec", [TINY, TINY.with_(Hq=8, Hkv=2, d=1024, ffn=1536, vocab=2048)])
def test_decode_logits_within_tolerance(spec, pack):
    """Prefill then teacher-forced decode steps through the paged decode path: logits vs
    the oracle.  Row-major weights (TMA boxes) and packed weights (bulk copies of
    pre-swizzled tiles; with PL_CHAIN=1 the persistent chain kernel, tests/test_chain_gpu.py)."""
    lens = [100, 37, 64]
    R, T = len(lens), sum(lens)
    steps = 5
    exe = StageExecutor(spec, 0, (0, spec.num_layers), True, True, torch.device("cuda", 0), seed=0,
                        pack_weights=pack,
                        max_tokens=T, max_reqs=R, max_ctx=256, num_blocks=3 * 4, n_slots=1)
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
    exe.stream.synchronize()

    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=256)
    caches = model.new_cache(R)
    toks = [torch.from_numpy(ids[cu[i]:cu[i + 1]]) for i in range(R)]
    ref = model.forward(toks, [torch.arange(n) for n in lens], caches)
    last_token = torch.zeros(R, dtype=torch.int64, device="cuda")
    worst = 0.0
    for k in range(steps):
        nxt = ref.argmax(-1)                         # teacher forcing with the oracle's tokens
        last_token.copy_(nxt)
        p = np.array([lens[i] + k for i in range(R)])
        dslots = rows[np.arange(R), p // 64] * 64 + p % 64
        meta = build_meta(R, R, mb_, p, dslots, np.arange(R), np.arange(R + 1), p + 1, np.arange(R), rows)
        exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
        torch.cuda.synchronize()
        exe.forward(0, R, R, True, 1, int(p.max()) + 1, last_token=last_token)
        exe.stream.synchronize()
        hn = ops.rmsnorm(exe.hidden[0][:R].clone(), exe.final_norm, spec.eps)
        got = OD.linear_acc(hn.cpu(), model.lm_head)
        ref = model.forward([nxt[i:i + 1] for i in range(R)], [torch.tensor([p[i]]) for i in range(R)], caches)
        err = (got - ref).abs().max().item()
        tol = tol_of(spec)
        worst = max(worst, err / tol)
        assert err <= tol, f"step {k}: max |dlogit| {err:.4f} (tol {tol:.4f})"
    exe.close()


@pytest.mark.parametrize("native", [True, False], ids=["native", "python"])
@pytest.mark.parametrize("S", [1, 4, 8])
def test_stage_counts_on_one_gpu(S, native):
    spec = TINY.with_(peaked=True, num_layers=max(4, S))
    cfg, cluster, plan, trace = config1(spec, S=S, n_req=5, in_len=70, out_len=9, mbt=256)
    res = run_gpu(spec, cfg, cluster, plan, trace, native=native)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy())


@pytest.mark.parametrize("native", [True, False], ids=["native", "python"])
def test_mixed_prefill_decode_microbatches(native):
    """allow_mixed_phase=True (engine.py:184-198): decoders and late-arriving prompts share
    micro-batches; schedule == pipelink's, tokens == the oracle's."""
    spec = TINY.with_(peaked=True)
    cluster = deploy.b200_cluster(2)
    plan = deploy.plan(cluster, spec, 2)
    ctrl = pipelink.ControllerConfig(max_batched_tokens=512, max_batch_size=8)
    cfg = deploy.engine_config(plan, spec, ctrl, chunk_size=4096, allow_mixed_phase=True)
    trace = pipelink.Trace(requests=[pipelink.Request(i, 0.0001 * i, 40 + 9 * i, 7) for i in range(8)])
    profiles = synth_profiles(plan)
    eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec, seed=0, native=native)
    res = eng.run(trace)
    ref = pipelink.PipelineEngine(cfg, cluster, profiles).run(trace)
    a, b = result_key(ref), result_key(res)
    for k in a:
        assert a[k] == b[k], f"schedule mismatch in {k}"
    phases = {mb[0] for mb in eng.gpu.mb_log}
    assert "mixed" in phases, f"trace produced no mixed micro-batch: {phases}"
    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=256)
    for r in trace.requests:
        want, _ = model.greedy([torch.from_numpy(prompt_tokens(0, r.id, r.input_len, spec.vocab))],
                               r.output_len)
        assert np.array_equal(res.b200.tokens[r.id], want[0].numpy()), f"request {r.id}"
    eng.close()


def test_prefill_chunking_on_and_off_same_tokens():
    """Chunk boundaries change only the transport, never the tokens (config 4 invariant)."""
    spec = TINY.with_(peaked=True)
    outs = []
    for chunk in (None, 4096):
        cfg, cluster, plan, trace = config1(spec, S=2, n_req=6, in_len=100, out_len=6, chunk=chunk)
        outs.append(run_gpu(spec, cfg, cluster, plan, trace).b200.tokens)
    for rid in outs[0]:
        assert np.array_equal(outs[0][rid], outs[1][rid])


def test_llama3_shape_truncated_tokens_identical():
    """Llama-3-8B widths (d=4096, GQA 32/8, ffn 14336, V=128256), 2 layers, 2 stages."""
    spec = LLAMA3_8B.with_(num_layers=2, peaked=True)
    cfg, cluster, plan, trace = config1(spec, S=2, n_req=4, in_len=96, out_len=6, mbt=512)
    res = run_gpu(spec, cfg, cluster, plan, trace)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy())


def test_qwen2_shape_truncated_tokens_identical():
    """Qwen2-72B widths (d=8192, GQA 64/8 -> group 8, qkv bias, ffn 29568, V=152064),
    2 layers, 2 stages: bias epilogues and the G=8 attention path end to end."""
    from paper_2507_05043_b200 import QWEN2_72B

    spec = QWEN2_72B.with_(num_layers=2, peaked=True)
    cfg, cluster, plan, trace = config1(spec, S=2, n_req=3, in_len=80, out_len=5, mbt=512)
    res = run_gpu(spec, cfg, cluster, plan, trace)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy()), f"request {r.id}"


def test_long_context_split_decode_attention_tokens_identical():
    """Prompts of 1100-1300 tokens: decode contexts exceed 1024, so each (request, kv head)
    splits into two items merged by the last arriver -- end to end through the pipeline."""
    spec = TINY.with_(peaked=True)
    cluster = deploy.b200_cluster(2)
    plan = deploy.plan(cluster, spec, 2)
    ctrl = pipelink.ControllerConfig(max_batched_tokens=4096, max_batch_size=4)
    cfg = deploy.engine_config(plan, spec, ctrl)
    trace = pipelink.Trace(requests=[pipelink.Request(i, 0.0, 1100 + 70 * i, 6) for i in range(4)])
    res = run_gpu(spec, cfg, cluster, plan, trace)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy()), f"request {r.id}"


@pytest.mark.parametrize("native", [True, False], ids=["native", "python"])
def test_link_throttle_replays_virtual_link_timing(native):
    """Throttle mode (transport.py:199-200 + engine.py:552 in wall time): every delivery is
    gated on the GPU clock at its virtual time, so the device run spans at least the virtual
    schedule's makespan (and not much more when compute is faster than the links), and the
    tokens are unchanged."""
    spec = TINY.with_(peaked=True)
    S = 2
    cluster = deploy.b200_cluster(S, 0.004, 2.0e6)     # 4 ms, 2 MB/s links
    plan = deploy.plan(cluster, spec, S)
    ctrl = pipelink.ControllerConfig(max_batched_tokens=256, max_batch_size=8)
    cfg = deploy.engine_config(plan, spec, ctrl, chunk_size=16384)
    trace = deploy.uniform_trace(4, 64, 5)
    profiles = synth_profiles(plan)
    eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec, throttle=True, native=native)
    res = eng.run(trace)
    ref = pipelink.PipelineEngine(cfg, cluster, profiles).run(trace)
    assert result_key(ref) == result_key(res)
    span = ref.end_ns / 1e9
    assert span > 0.05                                  # link-dominated schedule
    assert res.b200.run_time_s >= 0.97 * span, (res.b200.run_time_s, span)
    assert res.b200.run_time_s <= 1.5 * span + 0.05, (res.b200.run_time_s, span)
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy())
    eng.close()


def test_real_clock_run_result_feeds_reference_metrics():
    """RunResult on the device clock: summarize()/measure_bubble() apply unchanged."""
    spec = TINY.with_(peaked=True)
    cfg, cluster, plan, trace = config1(spec, S=2, n_req=6, in_len=64, out_len=8)
    res = run_gpu(spec, cfg, cluster, plan, trace)
    real = res.b200.real
    rep = pipelink.summarize(real.requests)
    assert rep.total_tokens == 6 * 8
    assert 0 < rep.ttft_p50_s <= rep.span_s <= res.b200.run_time_s + 1e-6
    for s in range(2):
        assert real.stage_busy_ns[s], "no real busy intervals"
        b = pipelink.measure_bubble(real, s, 0.0, real.end_ns / 1e9)
        assert 0.0 <= b < 1.0
    # per-request tokens are emitted in order on the device clock
    for rid, ts in res.b200.token_times_s.items():
        assert ts == sorted(ts) and len(ts) == 8


def test_realized_link_log_matches_virtual_chunks():
    """Per-chunk CUDA events on the link streams: the realized chunk sequence on every
    link is the LinkQueue's (same payloads, indices, sizes, order), chunks never overlap
    on a link, bytes are conserved and no chunk leaves before its payload exists."""
    spec = TINY.with_(peaked=True)
    cfg, cluster, plan, trace = config1(spec, S=2, n_req=6, in_len=300, out_len=5, chunk=16384)
    profiles = synth_profiles(plan)
    eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec)
    eng.gpu.record_links = True
    res = eng.run(trace)
    real = eng.gpu.realized_links
    for name in {e.link for e in res.link_events}:
        virt = [(e.payload_id, e.chunk_index, e.size_bytes) for e in res.link_events
                if e.link == name and e.event == "emit"]
        emits = [e for e in real if e.link == name and e.event == "emit"]
        sents = [e for e in real if e.link == name and e.event == "sent"]
        assert [(e.payload_id, e.chunk_index, e.size_bytes) for e in emits] == virt
        for a, b in zip(sents, emits[1:]):
            assert b.time_ns >= a.time_ns, "two chunks in flight on one link"
        enq = {e.payload_id: e.time_ns for e in real if e.link == name and e.event == "enqueue"}
        sizes = {}
        for e in emits:
            assert e.time_ns >= enq[e.payload_id] - 1000, "chunk left before its payload existed"
            sizes[e.payload_id] = sizes.get(e.payload_id, 0) + e.size_bytes
        virt_sizes = {e.payload_id: e.size_bytes for e in res.link_events
                      if e.link == name and e.event == "enqueue"}
        assert sizes == virt_sizes
    assert any(e.chunk_index > 0 for e in real), "prefill payloads were not chunked"
    eng.close()


def test_decode_rows_batch_invariant():
    """A decode request's result never depends on the decode micro-batch it rides in:
    every decode GEMM picks its split-K from the weight shape (N, K) only and the
    attention splits from the request's own context, so request 0's hidden row and
    greedy id are bit-identical at R = 1, 7, 64 and 200 (prefill micro-batches above 256
    tokens use the token-row orientation instead -- same bf16 rounding points, a
    different fp32 summation order -- so the claim is about decode)."""
    spec = LLAMA3_8B.with_(num_layers=2)
    R, L = 200, 24
    exe = StageExecutor(spec, 0, (0, 2), True, True, torch.device("cuda", 0), seed=0,
                        max_tokens=R * L, max_reqs=R, max_ctx=64, num_blocks=R, n_slots=1)
    rows = np.arange(R, dtype=np.int32)[:, None]
    lens = [L] * R
    cu = np.concatenate([[0], np.cumsum(lens)])
    pos = np.concatenate([np.arange(n) for n in lens])
    req_of = np.repeat(np.arange(R), lens)
    slots = rows[req_of, 0] * 64 + pos
    meta = build_meta(R * L, R, 1, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
    ids = np.concatenate([prompt_tokens(0, i, L, spec.vocab) for i in range(R)])
    exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
    exe.ids_dev[: R * L].copy_(torch.from_numpy(ids))
    torch.cuda.synchronize()
    exe.forward(0, R * L, R, False, L, L)
    exe.stream.synchronize()
    last = exe.out_ids[0][:R].clone()
    outs = []
    for n in (1, 7, 64, 200):
        p = np.full(n, L)
        meta = build_meta(n, n, 1, p, rows[:n, 0] * 64 + L, np.arange(n), np.arange(n + 1), p + 1,
                          np.arange(n), rows[:n])
        exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
        torch.cuda.synchronize()
        exe.forward(0, n, n, True, 1, L + 1, last_token=last)
        exe.stream.synchronize()
        outs.append((exe.hidden[0][0].clone().view(torch.int16).cpu(), int(exe.out_ids[0][0])))
    for h, t in outs[1:]:
        assert torch.equal(h, outs[0][0]) and t == outs[0][1]
    exe.close()


def test_fused_transport_same_tokens_and_link_log():
    """Fused transport (§8(f)3): decode payloads between stages of one process are stored
    by the producer's last residual epilogue straight into the next stage's buffer (no
    link copy).  Same schedule, same tokens as the copying transport and the oracle; the
    realized link log still follows the LinkQueue (tests/link_checks.py), decode chunks
    now zero-length at the producer's completion."""
    from link_checks import check_realized_link

    spec = TINY.with_(peaked=True, num_layers=4)
    cfg, cluster, plan, trace = config1(spec, S=4, n_req=6, in_len=90, out_len=7, mbt=256, chunk=4096)
    profiles = synth_profiles(plan)
    outs = {}
    for fuse in (False, True):
        eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec, fuse_transport=fuse)
        eng.gpu.record_links = True
        res = eng.run(trace)
        assert result_key(res) == result_key(pipelink.PipelineEngine(cfg, cluster, profiles).run(trace))
        for lp in eng.link_profiles:
            check_realized_link(eng.gpu.realized_links, res.link_events, lp.name)
        outs[fuse] = res.b200.tokens
        eng.close()
    _, _, want = oracle_greedy(spec, trace)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(outs[True][r.id], outs[False][r.id])
        assert np.array_equal(outs[True][r.id], want[i].numpy())
