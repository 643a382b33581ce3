"""Runtime monitoring: online StageProfile / LinkProfile estimates for the controller.

MoLink profiles stages and links at startup and keeps monitoring them while serving
(the reference leaves it as an open question, and
its live head loop, demo.py:125-184, plans with fixed profiles).  ``RuntimeMonitor``
collects measured samples while the live pipeline runs and, every ``epoch``
micro-batches, rebuilds the reference's own profile types so the unchanged
``choose_n`` plans with what the hardware is doing now:

* stage samples ``(stage, phase, batched_tokens, seconds)`` -- device-clock forward
  durations (CUDA events) that every stage reports for its last completed forward;
  per (stage, phase) and power-of-two token bucket the median of the last ``window``
  samples becomes a ``StageProfile`` point; points are made non-decreasing in tokens
  and every phase keeps >= 2 points (the startup profile fills missing buckets), the
  validity rules of profiles.py:38-64;
* round-trip samples ``(bytes per hop, seconds)`` of whole micro-batches (dispatch
  to token feedback on the head's wall clock) minus the stages' compute give the
  time on the S hops; one-way latency = the low quantile of those per-hop times at
  small payloads, bandwidth = bytes / (time - latency) over large payloads --
  ``LinkProfile(latency_s, bandwidth_bps)`` (profiles.py:75-92) for every hop.
"""

from __future__ import annotations

import math
from collections import defaultdict, deque

from ._pipelink import pipelink

Phase = pipelink.Phase


def _bucket(tokens: int) -> int:
    return 1 << max(0, math.ceil(math.log2(max(1, tokens))))


def _median(xs):
    s = sorted(xs)
    n = len(s)
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


class RuntimeMonitor:
    def __init__(self, stage_profiles, link_profiles, *, epoch: int = 32, window: int = 16,
                 small_bytes: int = 1 << 16, large_bytes: int = 1 << 20):
        self.base_stages = list(stage_profiles)
        self.base_links = list(link_profiles)
        self.stage_profiles = list(stage_profiles)
        self.link_profiles = list(link_profiles)
        self.epoch, self.window = epoch, window
        self.small, self.large = small_bytes, large_bytes
        self._stage = defaultdict(lambda: deque(maxlen=window))   # (s, phase, bucket) -> seconds
        self._hops = deque(maxlen=8 * window)                      # (bytes per hop, seconds per hop)
        self._since = 0
        self.updates = 0

    # ---------------------------------------------------------------- samples
    def stage_sample(self, stage: int, phase, tokens: int, seconds: float) -> None:
        if seconds > 0 and tokens > 0:
            self._stage[(stage, phase, _bucket(tokens))].append(seconds)

    def round_trip(self, bytes_per_hop: int, seconds: float, compute_s: float) -> None:
        """One micro-batch: dispatch -> feedback `seconds`, of which `compute_s` were the
        stages' forwards; the rest is spread over the S hops."""
        S = max(1, len(self.base_links))
        per_hop = (seconds - compute_s) / S
        if per_hop > 0:
            self._hops.append((bytes_per_hop, per_hop))

    def tick(self) -> bool:
        """One micro-batch finished; rebuild the profiles at each epoch boundary.
        Returns True when new profiles are in place."""
        self._since += 1
        if self._since < self.epoch:
            return False
        self._since = 0
        self.stage_profiles = [self._stage_profile(s, p) for s, p in enumerate(self.base_stages)]
        self.link_profiles = self._links()
        self.updates += 1
        return True

    # ------------------------------------------------------------- rebuilding
    def _stage_profile(self, s: int, base):
        entries = {}
        for phase in base.phases():
            pts = dict(base.points(phase))
            measured = {b: _median(v) for (st, ph, b), v in self._stage.items() if st == s and ph == phase and v}
            pts.update(measured)                       # measured buckets replace startup points
            prev = 0.0
            for tokens in sorted(pts):
                prev = max(prev, pts[tokens])          # non-decreasing in tokens (profiles.py:58-63)
                entries[(phase, tokens)] = prev
        return pipelink.StageProfile(stage_id=base.stage_id, layers=base.layers, entries=entries)

    def _links(self):
        if len(self._hops) < 4:
            return list(self.link_profiles)
        small = sorted(t for b, t in self._hops if b <= self.small)
        lat = small[len(small) // 10] if small else min(t for _, t in self._hops)
        bws = [b / (t - lat) for b, t in self._hops if b >= self.large and t > lat]
        out = []
        for lp in self.base_links:
            bw = _median(bws) if bws else lp.bandwidth_bps
            out.append(pipelink.LinkProfile(lp.src, lp.dst, max(0.0, lat), max(bw, 1.0)))
        return out
