"""RuntimeMonitor (runtime monitoring): profiles rebuilt from samples
are valid reference profiles and follow what was measured."""

import pipelink

from paper_2507_05043_b200.monitor import RuntimeMonitor

Phase = pipelink.Phase


def base():
    st = [pipelink.synth_profile(4, 1e-6, 2e-5, stage_id=i) for i in range(2)]
    ln = [pipelink.LinkProfile("a", "b", 2e-6, 9e11), pipelink.LinkProfile("b", "a", 2e-6, 9e11)]
    return st, ln


def test_epoch_rebuild_uses_measured_buckets_and_stays_valid():
    st, ln = base()
    m = RuntimeMonitor(st, ln, epoch=4, window=8)
    for _ in range(3):
        m.stage_sample(0, Phase.DECODE, 8, 3e-4)
        m.stage_sample(0, Phase.DECODE, 64, 2e-4)      # noisy: lower than 8 tokens
        m.stage_sample(1, Phase.PREFILL, 500, 5e-3)
        assert not m.tick()
    assert m.tick() and m.updates == 1
    p0 = dict(m.stage_profiles[0].points(Phase.DECODE))
    assert p0[8] == 3e-4 and p0[64] >= 3e-4           # measured, then made non-decreasing
    assert dict(m.stage_profiles[1].points(Phase.PREFILL))[512] == 5e-3
    for p in m.stage_profiles:                          # StageProfile validation passed
        assert all(len(p.points(ph)) >= 2 for ph in p.phases())


def test_links_from_round_trips():
    st, ln = base()
    m = RuntimeMonitor(st, ln, epoch=1, small_bytes=1 << 16, large_bytes=1 << 20)
    # two hops per round trip: small payloads show latency 10 us, large ones 1 MB / 100 GB/s more
    for _ in range(20):
        m.round_trip(4096, 2 * 10e-6 + 1e-3, 1e-3)
        m.round_trip(8 << 20, 2 * (10e-6 + (8 << 20) / 100e9) + 1e-3, 1e-3)
    m.tick()
    for lp in m.link_profiles:
        assert abs(lp.latency_s - 10e-6) < 1e-6
        assert abs(lp.bandwidth_bps / 100e9 - 1) < 0.02
    # the controller accepts the monitor's profiles
    cfg = pipelink.ControllerConfig(max_batched_tokens=512, max_batch_size=8)
    d = pipelink.choose_n(cfg, m.stage_profiles, m.link_profiles, 64, Phase.DECODE, bytes_per_token=512)
    assert d.n_microbatches >= 1
