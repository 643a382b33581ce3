"""Native scheduler parity: csrc/sched.cu == pipelink.PipelineEngine, bit for bit.

The C++ event loop (sched.cu) restates engine.py:264-600, controller.py:68-186,
transport.py:32-160 and profiles.py:95-121.  On randomized pipelines the
RunResult rebuilt from its logs (native.NativeScheduler) must equal the
unmodified reference engine's: events, link log, decisions, busy intervals,
emissions, request lifecycles.  Host-only -- no GPU needed.
"""

import random

import pytest

import pipelink
from pipelink import (
    ControllerConfig,
    EngineConfig,
    PipelineEngine,
    Trace,
    generate_trace,
    synth_profile,
)
from pipelines import decode_trace, uniform_pipeline
from test_driver_parity import random_setup, result_key

from paper_2507_05043_b200.native import NativeScheduler


def links_of(cfg, cluster):
    names = cfg.partition.node_names()
    if len(names) < 2:
        return []
    return [cluster.link(a, b) for a, b in list(zip(names, names[1:])) + [(names[-1], names[0])]]


def assert_native_same(cfg, cluster, profiles, trace, horizon=None):
    ref = PipelineEngine(cfg, cluster, profiles).run(trace, horizon_s=horizon)
    got = NativeScheduler(cfg, profiles, links_of(cfg, cluster)).run(trace, horizon_s=horizon)
    a, b = result_key(ref), result_key(got)
    for k in a:
        assert a[k] == b[k], f"mismatch in {k}"
    return ref


@pytest.mark.parametrize("seed", range(80))
def test_randomized_pipelines_match_reference(seed):
    rng = random.Random(1000 + seed)
    cfg, cluster, profiles, trace = random_setup(rng)
    assert_native_same(cfg, cluster, profiles, trace)


@pytest.mark.parametrize("seed", range(6))
def test_choose_n_matches_reference(seed):
    rng = random.Random(77 + seed)
    cfg, cluster, profiles, _ = random_setup(rng)
    links = links_of(cfg, cluster)
    sched = NativeScheduler(cfg, profiles, links)
    bpt = cfg.model.hidden_dim * cfg.model.dtype_bytes
    for _ in range(200):
        q = rng.choice([0, 1, 2, 7, 64, 333, 4096, 100000])
        ph = rng.choice([pipelink.Phase.PREFILL, pipelink.Phase.DECODE])
        want = pipelink.choose_n(cfg.controller, profiles, links, q, ph, bytes_per_token=bpt)
        assert sched.choose_n(q, ph) == want


def test_horizon_truncation_matches():
    cluster, model, plan, profiles = uniform_pipeline(3, 0.002, 0.001, hidden_dim=64, dtype_bytes=2)
    cfg = EngineConfig(partition=plan, model=model,
                       controller=ControllerConfig(max_batched_tokens=512, max_batch_size=8))
    assert_native_same(cfg, cluster, profiles, decode_trace(12), horizon=0.5)


def test_poisson_trace_matches():
    cluster, model, plan, profiles = uniform_pipeline(2, 0.001, 0.001, bandwidth=1e9, hidden_dim=64,
                                                      dtype_bytes=2)
    cfg = EngineConfig(partition=plan, model=model, chunk_size=4096,
                       controller=ControllerConfig(max_batched_tokens=256, max_batch_size=8))
    trace = Trace(requests=generate_trace(rate=100.0, duration=1.5, seed=17).requests[:100])
    assert assert_native_same(cfg, cluster, profiles, trace).all_finished


def test_eight_stage_weak_link_dynamic_matches():
    """The 8-stage throttled configuration (BASELINE config 5 shape) at full trace size."""
    cluster, model, plan, _ = uniform_pipeline(8, 0.002, 0.015, bandwidth=12.5e6,
                                               hidden_dim=4096, dtype_bytes=2)
    profiles = [synth_profile(1, 2e-6, 3e-4, i) for i in range(8)]
    cfg = EngineConfig(partition=plan, model=model, chunk_size=262_144,
                       controller=ControllerConfig(max_batched_tokens=2048, max_batch_size=64))
    trace = Trace(requests=[pipelink.Request(i, 0.001 * i, 128 + 37 * (i % 7), 16 + i % 9)
                            for i in range(64)])
    assert assert_native_same(cfg, cluster, profiles, trace).all_finished


def test_duplicate_request_id_raises_config_error():
    cluster, model, plan, profiles = uniform_pipeline(2, 0.001, 0.001, hidden_dim=64, dtype_bytes=2)
    cfg = EngineConfig(partition=plan, model=model,
                       controller=ControllerConfig(max_batched_tokens=256, max_batch_size=8))
    trace = Trace(requests=[pipelink.Request(1, 0.0, 8, 2), pipelink.Request(1, 0.0, 8, 2)])
    with pytest.raises(pipelink.ConfigError):
        NativeScheduler(cfg, profiles, links_of(cfg, cluster)).run(trace)
