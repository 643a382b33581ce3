"""Known answers of the reference's own test-suite, replayed through the B200 driver.

The scheduling / chunking / link-timing half of the hot path is pinned by the
reference tests' golden numbers.  Each case below restates one
known answer (cited) and checks it both on the installed, unmodified pipelink
(pinning the oracle we import) and through `PipelineDriver` (the schedule the
GPU backend executes).
"""

import pytest

import pipelink
from pipelink import (
    ControllerConfig,
    EngineConfig,
    LinkProfile,
    Payload,
    PayloadClass,
    Phase,
    choose_n,
    flat_profile,
    measure_bubble,
    predict_bubble,
    replay_link,
)
from pipelines import decode_trace, uniform_pipeline

from paper_2507_05043_b200.driver import PipelineDriver

s_to_ns = pipelink.transport.s_to_ns
transmission_ns = pipelink.transport.transmission_ns
first_emit_delay_ns = pipelink.transport.first_emit_delay_ns


def ring(S, lat, bw=1e18):
    names = [f"s{i}" for i in range(S)]
    return [LinkProfile(a, b, lat, bw) for a, b in list(zip(names, names[1:])) + [(names[-1], names[0])]]


def flats(S, sec):
    return [flat_profile(sec, stage_id=i) for i in range(S)]


# test_controller.py:31-39 -- 2 stages, 10 ms compute, 5 ms hops: bubble 1/3 at n=2, 0 at n=3
def test_desk_bubbles():
    assert predict_bubble(2, flats(2, 0.010), ring(2, 0.005), 4, Phase.DECODE) == pytest.approx(1 / 3)
    assert predict_bubble(3, flats(2, 0.010), ring(2, 0.005), 4, Phase.DECODE) == 0.0


# test_controller.py:73-78 -- desk case picks n=3 with budget 4
def test_desk_choice_through_driver_memo():
    cluster, model, plan, profiles = uniform_pipeline(2, 0.010, 0.005)
    cfg = EngineConfig(partition=plan, model=model,
                       controller=ControllerConfig(max_batched_tokens=12, max_batch_size=4), chunk_size=None)
    res = PipelineDriver(cfg, cluster, profiles).run(decode_trace(12), horizon_s=0.4)
    d = res.decisions[0][1]
    assert (d.n_microbatches, d.token_budget_per_microbatch, d.predicted_bubble_fraction) == (3, 4, 0.0)


# test_controller.py:104-119 -- minimality spot checks (S, hop/compute) -> n
@pytest.mark.parametrize("S,ratio,n", [(2, 0.25, 3), (3, 0.5, 5), (4, 1.0, 8)])
def test_minimality(S, ratio, n):
    cfg = ControllerConfig(max_batched_tokens=64, max_batch_size=64, n_max=2 * S)
    d = choose_n(cfg, flats(S, 0.010), ring(S, 0.010 * ratio), 64, Phase.DECODE)
    assert d.n_microbatches == n


# test_acceptance.py:103-126 -- dynamic n beats fixed n=S by +50%, utilisation 1.0 vs 2/3
def test_criterion_2_through_driver():
    def run(n_max):
        cluster, model, plan, profiles = uniform_pipeline(2, 0.010, 0.005)
        cfg = EngineConfig(partition=plan, model=model, chunk_size=None,
                           controller=ControllerConfig(max_batched_tokens=12, max_batch_size=4,
                                                       n_max=n_max))
        return PipelineDriver(cfg, cluster, profiles).run(decode_trace(12), horizon_s=0.4)

    fixed, dynamic = run(2), run(None)
    w0, w1 = 0.09, 0.39
    gain = dynamic.tokens_in_window(w0, w1) / fixed.tokens_in_window(w0, w1) - 1.0
    assert abs(gain - 0.50) <= 0.02
    assert abs((1 - measure_bubble(dynamic, 0, w0, w1)) - 1.0) <= 1e-9
    assert abs((1 - measure_bubble(fixed, 0, w0, w1)) - 2 / 3) <= 1e-9


# test_transport.py:57-63 -- 600,000-byte prefill in 256 KiB chunks: [262144, 262144, 75712]
def test_chunk_split_through_driver():
    S = 2
    cluster, _, plan, profiles = uniform_pipeline(S, 0.001, 0.0, bandwidth=1e9)
    model = pipelink.ModelSpec("wide", S, 75_000, 2, 1)   # 4 tokens x 150,000 B = 600,000 B
    cfg = EngineConfig(partition=plan, model=model, chunk_size=262_144,
                       controller=ControllerConfig(max_batched_tokens=4, max_batch_size=1))
    trace = pipelink.Trace(requests=[pipelink.Request(0, 0.0, 4, 1)])
    res = PipelineDriver(cfg, cluster, profiles).run(trace)
    emits = [e.size_bytes for e in res.link_events if e.event == "emit" and e.link == "b0->b1"]
    assert emits == [262_144, 262_144, 75_712]


# test_transport.py:238-240 -- 256 KiB at 100 Mbps takes 20,971,520 ns on the wire
def test_transmission_ns_golden():
    assert transmission_ns(LinkProfile("a", "b", 0.0, 12_500_000), 262_144) == 20_971_520


# test_transport.py:102-109 -- single unchunked 256 KiB payload delivered at 30.97152 ms
def test_delivery_time_golden():
    link = LinkProfile("a", "b", latency_s=0.010, bandwidth_bps=12_500_000)
    ev = replay_link(link, [(0, Payload(1, PayloadClass.PREFILL, 262_144, 1, 0))], chunk_size=None)
    assert [e.time_ns for e in ev if e.event == "deliver"] == [s_to_ns(0.03097152)]


# test_acceptance.py:132-154 -- chunking cuts the decode head-of-line wait 655.4 ms -> 20.97 ms
def test_criterion_3_chunking_golden():
    link = LinkProfile("a", "b", latency_s=0.010, bandwidth_bps=12_500_000)
    arrivals = [(0, Payload(0, PayloadClass.PREFILL, 1000 * 4096 * 2, 0, 0)),
                (0, Payload(1, PayloadClass.DECODE, 4 * 4096 * 2, 1, 0))]
    un = first_emit_delay_ns(replay_link(link, arrivals, chunk_size=None), 1)
    ch = first_emit_delay_ns(replay_link(link, arrivals, chunk_size=262_144), 1)
    assert un == 655_360_000 and ch == 20_971_520


# test_transport.py:66-73 -- decode arrival preempts at the next chunk boundary
def test_decode_preemption_order():
    q = pipelink.LinkQueue(chunk_size=100)
    q.enqueue(Payload(1, PayloadClass.PREFILL, 350, 1, 0))
    first = q.next_chunk()
    q.enqueue(Payload(2, PayloadClass.DECODE, 8, 2, 0))
    order = [(first.payload_id, first.index)]
    while (c := q.next_chunk()) is not None:
        order.append((c.payload_id, c.index))
    assert order == [(1, 0), (2, 0), (1, 1), (1, 2), (1, 3)]


# test_acceptance.py:160-181 -- zero transfers: n = S and utilisation 1.0 (S = 1..4)
@pytest.mark.parametrize("S", [1, 2, 3, 4])
def test_criterion_4_zero_transfer_identity_through_driver(S):
    cluster, model, plan, profiles = uniform_pipeline(S, 0.010, 0.0)
    cfg = EngineConfig(partition=plan, model=model, chunk_size=None,
                       controller=ControllerConfig(max_batched_tokens=4 * S, max_batch_size=4, n_max=16,
                                                   bubble_epsilon=0.0))
    res = PipelineDriver(cfg, cluster, profiles).run(decode_trace(4 * S), horizon_s=0.6)
    w0 = 2 * S * 0.010
    assert abs((1 - measure_bubble(res, 0, w0, w0 + 10 * S * 0.010)) - 1.0) <= 1e-9
