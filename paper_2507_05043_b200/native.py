"""Python face of the native scheduler (csrc/sched.cu) and pipeline runtime (csrc/runtime.cu).

``NativeScheduler`` holds one ``pl_sched`` handle built from the reference's
own configuration objects (EngineConfig / StageProfile / LinkProfile) and turns
the C++ logs back into a reference ``RunResult`` -- so ``measure_bubble``,
``summarize`` and the parity tests read it unchanged.  The event loop, the
controller search and the link queues run in C++; Python only converts.

    sched = NativeScheduler(cfg, stage_profiles, link_profiles)
    result = sched.run(trace)                     # == pipelink.PipelineEngine(...).run(trace)
    result = sched.run(trace, pipeline=handle)    # same schedule, GPU work issued natively
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from ._pipelink import pipelink

E = pipelink.engine
T_ = pipelink.transport
EventKind = E.EventKind
RequestState = pipelink.RequestState
PayloadClass = T_.PayloadClass
Phase = pipelink.Phase
NS = T_.NS_PER_S
FEEDBACK_BYTES = pipelink.placement.TOKEN_FEEDBACK_BYTES

_STATES = (RequestState.QUEUED, RequestState.PREFILL, RequestState.DECODING, RequestState.FINISHED)
_CLASSES = (PayloadClass.PREFILL, PayloadClass.DECODE)
_LINK_EVENTS = ("enqueue", "emit", "sent", "deliver")
_KINDS = {int(k): k for k in EventKind}


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def _chunk_size(cs) -> int:
    if cs is None or (isinstance(cs, float) and math.isinf(cs)):
        return -1
    return int(cs)


class LazyRunResult(E.RunResult):
    """RunResult whose event and link logs become Python objects on first access
    (hundreds of thousands of rows on long runs; most callers never read them)."""

    def __init__(self, *, events_fn, link_events_fn, **kw):
        self._events_fn, self._link_events_fn = events_fn, link_events_fn
        self._ev = self._lk = None
        super().__init__(events=None, link_events=None, **kw)

    @property
    def events(self):
        if self._ev is None and self._events_fn is not None:
            self._ev, self._events_fn = self._events_fn(), None
        return self._ev

    @events.setter
    def events(self, v):
        if v is not None:
            self._ev, self._events_fn = v, None

    @property
    def link_events(self):
        if self._lk is None and self._link_events_fn is not None:
            self._lk, self._link_events_fn = self._link_events_fn(), None
        return self._lk

    @link_events.setter
    def link_events(self, v):
        if v is not None:
            self._lk, self._link_events_fn = v, None


class NativeScheduler:
    def __init__(self, cfg, stage_profiles, link_profiles, bytes_per_token: int | None = None):
        S = len(stage_profiles)
        ctrl = cfg.controller
        self.cfg = cfg
        self.stage_profiles = list(stage_profiles)
        self.link_profiles = list(link_profiles)
        self.S = S
        off, xs, ys = [0], [], []
        for p in stage_profiles:
            for ph in (Phase.PREFILL, Phase.DECODE):
                pts = p.points(ph)
                xs += [int(t) for t, _ in pts]
                ys += [float(v) for _, v in pts]
                off.append(len(xs))
        self._keep = {
            "off": np.asarray(off, dtype=np.int64), "x": np.asarray(xs, dtype=np.int64),
            "y": np.asarray(ys, dtype=np.float64),
            "lat": np.asarray([lp.latency_s for lp in link_profiles], dtype=np.float64),
            "bw": np.asarray([lp.bandwidth_bps for lp in link_profiles], dtype=np.float64),
        }
        k = self._keep
        c = N.SchedConfig()
        c.n_stages, c.n_links = S, len(link_profiles)
        c.max_batched_tokens, c.max_batch_size = ctrl.max_batched_tokens, ctrl.max_batch_size
        c.n_max = ctrl.effective_n_max(S)
        c.bubble_epsilon, c.gain_delta = ctrl.bubble_epsilon, ctrl.gain_delta
        c.fixed_compute = int(ctrl.mode is pipelink.controller.BudgetMode.FIXED_COMPUTE)
        c.decision_stride = ctrl.decision_stride
        c.chunk_size = _chunk_size(cfg.chunk_size)
        c.fcfs = int(cfg.scheduling_policy is E.SchedulingPolicy.FCFS)
        c.allow_mixed = int(bool(cfg.allow_mixed_phase))
        c.bytes_per_token = (bytes_per_token if bytes_per_token is not None
                             else cfg.model.hidden_dim * cfg.model.dtype_bytes)
        c.feedback_bytes = FEEDBACK_BYTES
        c.prof_off, c.prof_x, c.prof_y = _ptr(k["off"]), _ptr(k["x"]), _ptr(k["y"])
        c.link_latency_s, c.link_bandwidth = _ptr(k["lat"]), _ptr(k["bw"])
        h = C.c_void_p()
        N.check(N.lib().pl_sched_create(C.byref(c), C.byref(h)), "pl_sched_create")
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().pl_sched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def choose_n(self, queued_tokens: int, phase) -> "pipelink.ControllerDecision":
        n, b, bub = C.c_int32(), C.c_int64(), C.c_double()
        N.check(N.lib().pl_sched_choose_n(self._h, int(queued_tokens), 1 if phase is Phase.DECODE else 0,
                                          C.byref(n), C.byref(b), C.byref(bub)), "pl_sched_choose_n")
        return pipelink.ControllerDecision(n.value, b.value, bub.value)

    # ---------------------------------------------------------------- run
    def run(self, trace, horizon_s: float | None = None, pipeline=None):
        seen = set()
        rows = np.empty((len(trace.requests), 4), dtype=np.int64)
        for i, r in enumerate(trace.requests):
            if r.id in seen:
                raise pipelink.ConfigError(f"duplicate request id {r.id} in trace")
            seen.add(r.id)
            rows[i] = (r.id, T_.s_to_ns(r.arrival_time), r.input_len, r.output_len)
        horizon = -1 if horizon_s is None else T_.s_to_ns(horizon_s)
        N.check(N.lib().pl_sched_run(self._h, _ptr(rows), len(rows), horizon, pipeline), "pl_sched_run")
        return self._result(trace)

    def _result(self, trace):
        lib = N.lib()
        cnt = np.zeros(8, dtype=np.int64)
        N.check(lib.pl_sched_counts(self._h, _ptr(cnt)), "pl_sched_counts")
        ne, nl, nd, nem, nfc, nb, end_ns, all_fin = (int(x) for x in cnt)
        nr = len(trace.requests)
        ev = np.zeros((ne, 4), dtype=np.int64)
        lk = np.zeros((nl, 7), dtype=np.int64)
        de = np.zeros((nd, 3), dtype=np.int64)
        bu = np.zeros(nd, dtype=np.float64)
        em = np.zeros((nem, 2), dtype=np.int64)
        fc = np.zeros((nfc, 2), dtype=np.int64)
        busy = np.zeros((nb, 3), dtype=np.int64)
        rs = np.zeros((nr, 2), dtype=np.int64)
        rt = np.zeros((nr, 2), dtype=np.float64)
        N.check(lib.pl_sched_read(self._h, _ptr(ev), _ptr(lk), _ptr(de), _ptr(bu), _ptr(em), _ptr(fc),
                                  _ptr(busy), _ptr(rs), _ptr(rt)), "pl_sched_read")
        kinds = _KINDS
        names = [lp.name for lp in self.link_profiles]

        def events():
            return [E.EngineEvent(t, kinds[k], s, st) for t, k, s, st in ev.tolist()]

        def link_events():
            return [T_.LinkEvent(t, names[li], p, i, sz, _CLASSES[c], _LINK_EVENTS[e])
                    for t, li, p, i, sz, c, e in lk.tolist()]

        decisions = [(it, pipelink.ControllerDecision(n, b, x))
                     for (it, n, b), x in zip(de.tolist(), bu.tolist())]
        stage_busy = [[] for _ in range(self.S)]
        for s, a, b in busy.tolist():
            stage_busy[s].append((a, b))
        reqs = []
        for r, (state, tok), (ft, fin) in zip(trace.requests, rs.tolist(), rt.tolist()):
            c = r.fresh_copy()
            c.arrival_time = T_.s_to_ns(r.arrival_time) / NS
            c.state = _STATES[state]
            c.tokens_emitted = tok
            c.first_token_time = None if math.isnan(ft) else ft
            c.finish_time = None if math.isnan(fin) else fin
            reqs.append(c)
        reqs.sort(key=lambda q: q.id)
        return LazyRunResult(
            events_fn=events, link_events_fn=link_events, requests=reqs, decisions=decisions,
            stage_busy_ns=stage_busy, token_emissions=[tuple(x) for x in em.tolist()],
            first_compute_ns={rid: t for rid, t in fc.tolist()}, end_ns=end_ns, all_finished=bool(all_fin))
