"""Schedule parity: the B200 driver's decisions equal the reference engine's, bit for bit.

`PipelineDriver.run` (no backend work) vs the unmodified
`pipelink.PipelineEngine.run` (engine.py:509-600) on randomized pipelines:
event log, link log (chunk boundaries, emit/sent/deliver times), controller
decisions, busy intervals, token emissions and per-request lifecycles must be
identical.  With a GPU backend attached the driver makes the same decisions
(decisions never read a wall clock), so these logs are the schedule/chunk
parity proof for real runs too.
"""

import random

import pytest

import pipelink
from pipelink import (
    ClusterSpec,
    ControllerConfig,
    EngineConfig,
    LinkProfile,
    PartitionPlan,
    PipelineEngine,
    Request,
    SchedulingPolicy,
    Trace,
    flat_profile,
    generate_trace,
    synth_profile,
)
from pipelines import decode_trace, make_node, uniform_pipeline

from paper_2507_05043_b200.driver import PipelineDriver
from paper_2507_05043_b200.spec import TINY, LLAMA3_8B


def result_key(res):
    from paper_2507_05043_b200.engine import schedule_key

    return schedule_key(res)


def assert_same(cfg, cluster, profiles, trace, horizon=None):
    ref = PipelineEngine(cfg, cluster, profiles).run(trace, horizon_s=horizon)
    got = PipelineDriver(cfg, cluster, profiles).run(trace, horizon_s=horizon)
    a, b = result_key(ref), result_key(got)
    for k in a:
        assert a[k] == b[k], f"mismatch in {k}"
    return ref


def random_setup(rng: random.Random):
    S = rng.choice([1, 2, 2, 3, 4, 8])
    names = [f"n{i}" for i in range(S)]
    nodes = {n: make_node(n) for n in names}
    links = {}
    if S > 1:
        for src, dst in list(zip(names, names[1:])) + [(names[-1], names[0])]:
            links[(src, dst)] = LinkProfile(src, dst, rng.choice([0.0, 2e-6, 1e-3, 0.015]),
                                            rng.choice([9e11, 1.25e7, 1e9, 5e7]))
    cluster = ClusterSpec(nodes=nodes, links=links)
    L = S * rng.randint(1, 3)
    model = pipelink.ModelSpec("m", L, rng.choice([64, 256, 4096]), 2, 1)
    per = L // S
    plan = PartitionPlan(stages=tuple((names[i], (i * per, (i + 1) * per)) for i in range(S)),
                         head=names[0])
    profiles = []
    for i in range(S):
        if rng.random() < 0.5:
            profiles.append(synth_profile(per, rng.uniform(1e-6, 1e-4), rng.uniform(1e-5, 1e-3), i))
        else:
            profiles.append(flat_profile(rng.uniform(1e-4, 1e-2), i, per))
    ctrl = ControllerConfig(
        max_batched_tokens=rng.choice([64, 256, 2048, 32768]),
        max_batch_size=rng.choice([1, 4, 8, 64]),
        n_max=rng.choice([None, 1, S, 2 * S + 1]),
        decision_stride=rng.choice([1, 1, 3]),
    )
    cfg = EngineConfig(partition=plan, model=model, controller=ctrl,
                       chunk_size=rng.choice([None, 4096, 262_144]),
                       scheduling_policy=rng.choice(list(SchedulingPolicy)),
                       allow_mixed_phase=rng.random() < 0.3)
    n = rng.randint(1, 40)
    reqs, t = [], 0.0
    for i in range(n):
        t += rng.choice([0.0, 0.0, rng.uniform(0, 0.01)])
        reqs.append(Request(id=i, arrival_time=t, input_len=rng.randint(1, 700),
                            output_len=rng.randint(1, 20)))
    return cfg, cluster, profiles, Trace(requests=reqs)


@pytest.mark.parametrize("seed", range(40))
def test_randomized_pipelines_match_reference(seed):
    rng = random.Random(1000 + seed)
    cfg, cluster, profiles, trace = random_setup(rng)
    assert_same(cfg, cluster, profiles, trace)


def test_horizon_truncation_matches():
    cluster, model, plan, profiles = uniform_pipeline(3, 0.002, 0.001, hidden_dim=64, dtype_bytes=2)
    cfg = EngineConfig(partition=plan, model=model,
                       controller=ControllerConfig(max_batched_tokens=512, max_batch_size=8))
    assert_same(cfg, cluster, profiles, decode_trace(12), horizon=0.5)


def test_poisson_trace_matches():
    cluster, model, plan, profiles = uniform_pipeline(2, 0.001, 0.001, bandwidth=1e9, hidden_dim=64,
                                                      dtype_bytes=2)
    cfg = EngineConfig(partition=plan, model=model, chunk_size=4096,
                       controller=ControllerConfig(max_batched_tokens=256, max_batch_size=8))
    trace = Trace(requests=generate_trace(rate=100.0, duration=1.5, seed=17).requests[:100])
    ref = assert_same(cfg, cluster, profiles, trace)
    assert ref.all_finished


@pytest.mark.parametrize("spec", [TINY, LLAMA3_8B])
def test_payload_sizing_is_bf16_residual_stream(spec):
    """engine.py:406 sizes the forward payload T*hidden_dim*dtype_bytes: with the
    DecoderSpec's ModelSpec that is exactly one bf16 [T, d] residual stream."""
    m = spec.model_spec()
    assert m.activation_bytes(17) == 17 * spec.d * 2
    assert m.bytes_per_layer == spec.layer_bytes()
