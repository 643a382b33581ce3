"""Virtual-clock pipeline driver: the reference's scheduling semantics, real work hooks.

The reference engine (pipelink/engine.py:241-600) decides everything on an
integer-nanosecond virtual clock and *simulates* the two hot-path subsystems.
This driver makes exactly the same decisions -- same heap tie order
(engine.py:42-49), same boundary rule (engine.py:456-505), same payload sizing
(engine.py:390-418), same link mechanics (engine.py:347-372, 546-576), same
token accounting (engine.py:422-442) -- by calling the reference's unchanged
``choose_n``, ``admit_and_batch``, ``LinkQueue``, ``compute_time`` and
``transmission_ns``, and it reports a reference ``RunResult`` so ``measure_bubble``
and ``summarize`` apply unchanged.  What differs is that every decision also
fires a backend hook that issues the real work:

  hook                      reference site          B200 backend action
  ------------------------  ----------------------  ----------------------------------------
  admit(mb)                 engine.py:481-504       build KV block tables / metadata
  compute(stage, mb)        engine.py:384           pl_stage_forward on the stage's stream
  emit(link, chunk, off)    engine.py:347-356       one NCCL send/recv (or peer copy) of
                                                    bytes [off, off+size) of the payload
  delivered(link, mb)       engine.py:560-576       return hop lands: token scatter on head
  feedback(mb)              engine.py:422-442       release the micro-batch slot

Because decisions never depend on wall-clock completions, the schedule, the
chunk boundaries and the token accounting are bit-identical to
``PipelineEngine.run`` for the same profiles (tests/test_driver_parity.py);
the GPU executes the resulting DAG asynchronously in per-stage FIFO order.

``choose_n`` is pure in (profiles, links, demand, phase) for a fixed run, so
the driver memoizes it (SURVEY hard part 3): the unchanged Python search costs
19-760 us per call, comparable to a B200 stage step.
"""

from __future__ import annotations

import heapq
from collections import deque
from dataclasses import dataclass, field

from ._pipelink import pipelink

E = pipelink.engine
T_ = pipelink.transport
EventKind = E.EventKind
BatchPhase = E.BatchPhase
EngineEvent = E.EngineEvent
LinkEvent = T_.LinkEvent
Payload = T_.Payload
PayloadClass = T_.PayloadClass
RequestState = pipelink.RequestState
Phase = pipelink.Phase
NS = T_.NS_PER_S
s_to_ns = T_.s_to_ns
transmission_ns = T_.transmission_ns
compute_time = pipelink.compute_time
FEEDBACK_BYTES = pipelink.placement.TOKEN_FEEDBACK_BYTES

_ARRIVAL, _BOUNDARY, _DONE, _SENT, _DELIVERED = (
    int(EventKind.ARRIVAL), int(EventKind.ITERATION_BOUNDARY), int(EventKind.COMPUTE_DONE),
    int(EventKind.CHUNK_SENT), int(EventKind.PAYLOAD_DELIVERED))


class Backend:
    """No-op hooks (pure virtual run).  Subclasses issue real work."""

    def start(self, driver: "PipelineDriver", trace) -> None: ...
    def admit(self, mb, now_ns: int) -> None: ...
    def compute(self, stage: int, mb, now_ns: int) -> None: ...
    def emit(self, link: int, payload, chunk, offset: int, now_ns: int) -> None: ...
    def delivered(self, link: int, payload, mb, now_ns: int) -> None: ...
    def feedback(self, mb, now_ns: int) -> None: ...
    def finish(self, result) -> None: ...


@dataclass
class _StageState:
    idx: int
    profile: object
    busy: bool = False
    current: object = None
    started: int = 0
    waiting: deque = field(default_factory=deque)
    intervals: list = field(default_factory=list)


@dataclass
class _LinkState:
    idx: int
    profile: object
    queue: object
    dst: int
    is_return: bool
    busy: bool = False
    owner: dict = field(default_factory=dict)   # payload id -> micro-batch
    sent_bytes: dict = field(default_factory=dict)  # payload id -> bytes already chunked out
    payloads: dict = field(default_factory=dict)


class PipelineDriver:
    """Drop-in for ``pipelink.PipelineEngine(cfg, cluster, stage_profiles)`` whose
    ``run(trace)`` returns the identical ``RunResult`` while a backend does the work."""

    def __init__(self, cfg, cluster, stage_profiles, backend: Backend | None = None):
        names = cfg.partition.node_names()
        if len(stage_profiles) != len(names):
            raise pipelink.ConfigError(
                f"{len(names)} stages in plan but {len(stage_profiles)} profiles")
        for n in names:
            if n not in cluster.nodes:
                raise pipelink.ConfigError(f"plan references unregistered node {n}")
        hops = list(zip(names, names[1:])) + [(names[-1], names[0])] if len(names) > 1 else []
        links = []
        for src, dst in hops:
            lp = cluster.link(src, dst)
            if lp is None:
                raise pipelink.ConfigError(f"cluster is missing required link {src}->{dst}")
            links.append(lp)
        self.cfg = cfg
        self.cluster = cluster
        self.stage_profiles = list(stage_profiles)
        self.link_profiles = links
        self.bytes_per_token = cfg.model.hidden_dim * cfg.model.dtype_bytes
        self.backend = backend or Backend()
        self._decision_cache: dict = {}
        self._compute_ns_cache: dict = {}

    def set_link_profiles(self, link_profiles) -> None:
        """Swap in measured link estimates (forward hops + return hop, cluster order)."""
        if len(link_profiles) != len(self.link_profiles):
            raise pipelink.ConfigError("link profile count must equal the hop count")
        self.link_profiles = list(link_profiles)
        self._decision_cache.clear()

    def set_stage_profiles(self, stage_profiles) -> None:
        """Swap in measured profiles (startup profiling) before the next run."""
        if len(stage_profiles) != len(self.stage_profiles):
            raise pipelink.ConfigError("profile count must equal the stage count")
        self.stage_profiles = list(stage_profiles)
        self._decision_cache.clear()
        self._compute_ns_cache.clear()

    # --------------------------------------------------------------- helpers
    def _post(self, t: int, kind: int, subject: int, data=None) -> None:
        heapq.heappush(self._heap, (t, kind, subject, self._seq, data))
        self._seq += 1

    def _note(self, t: int, kind, subject: int, stage: int = -1) -> None:
        self._events.append(EngineEvent(t, kind, subject, stage))

    def _note_link(self, ln: _LinkState, t: int, pid: int, idx: int, size: int, pclass, what: str):
        self._link_log.append(LinkEvent(t, ln.profile.name, pid, idx, size, pclass, what))

    def _compute_ns(self, st: _StageState, phase, tokens: int) -> int:
        key = (st.idx, phase, tokens)
        ns = self._compute_ns_cache.get(key)
        if ns is None:
            ns = max(1, s_to_ns(compute_time(st.profile, phase, tokens)))
            self._compute_ns_cache[key] = ns
        return ns

    def _decide(self, phase):
        demand = len(self._ready) + sum(m.batched_tokens for m in self._inflight.values()) \
            + sum(r.input_len for r in self._pending)
        key = (demand, phase)
        d = self._decision_cache.get(key)
        if d is None:
            d = pipelink.choose_n(self.cfg.controller, self.stage_profiles, self.link_profiles,
                                  demand, phase, bytes_per_token=self.bytes_per_token)
            self._decision_cache[key] = d
        return d

    # ------------------------------------------------------------- stages
    def _launch_compute(self, st: _StageState, now: int) -> None:
        if st.busy or not st.waiting:
            return
        mb = st.waiting.popleft()
        st.busy, st.current, st.started = True, mb, now
        phase = Phase.DECODE if mb.phase is BatchPhase.DECODE else Phase.PREFILL
        dur = self._compute_ns(st, phase, mb.batched_tokens)
        if st.idx == 0:
            for rid in mb.request_ids:
                self._first_compute.setdefault(rid, now)
        self._post(now + dur, _DONE, mb.id, st.idx)
        self.backend.compute(st.idx, mb, now)

    def _compute_finished(self, s: int, mb_id: int, now: int) -> None:
        st = self._stages[s]
        mb = st.current
        assert mb is not None and mb.id == mb_id
        st.intervals.append((st.started, now))
        st.busy, st.current = False, None
        self._note(now, EventKind.COMPUTE_DONE, mb.id, s)
        if s < len(self._stages) - 1:
            pclass = PayloadClass.DECODE if mb.phase is BatchPhase.DECODE else PayloadClass.PREFILL
            self._enqueue(self._links[s], mb, max(1, mb.batched_tokens * self.bytes_per_token), pclass, now)
        elif self._links:
            self._enqueue(self._links[-1], mb, max(1, FEEDBACK_BYTES * len(mb.request_ids)),
                          PayloadClass.DECODE, now)
        else:  # single stage: tokens surface at compute completion
            self._emit_tokens(mb, now)
            self._want_boundary(now)
        self._launch_compute(st, now)
        if s == 0:
            self._want_boundary(now)

    # -------------------------------------------------------------- links
    def _enqueue(self, ln: _LinkState, mb, size: int, pclass, now: int) -> None:
        p = Payload(id=self._next_payload, phase_class=pclass, size_bytes=size,
                    micro_batch_id=mb.id, enqueue_time=now)
        self._next_payload += 1
        ln.owner[p.id] = mb
        ln.payloads[p.id] = p
        ln.sent_bytes[p.id] = 0
        ln.queue.enqueue(p)
        self._note_link(ln, now, p.id, -1, size, pclass, "enqueue")
        if not ln.busy:
            self._pump(ln, now)

    def _pump(self, ln: _LinkState, now: int) -> None:
        ch = ln.queue.next_chunk()
        if ch is None:
            ln.busy = False
            return
        ln.busy = True
        self._note_link(ln, now, ch.payload_id, ch.index, ch.size_bytes, ch.phase_class, "emit")
        self._post(now + transmission_ns(ln.profile, ch.size_bytes), _SENT, ch.payload_id, (ln.idx, ch))
        off = ln.sent_bytes[ch.payload_id]
        ln.sent_bytes[ch.payload_id] = off + ch.size_bytes
        self.backend.emit(ln.idx, ln.payloads[ch.payload_id], ch, off, now)

    def _chunk_sent(self, link_idx: int, ch, now: int) -> None:
        ln = self._links[link_idx]
        self._note_link(ln, now, ch.payload_id, ch.index, ch.size_bytes, ch.phase_class, "sent")
        self._note(now, EventKind.CHUNK_SENT, ch.payload_id, -1)
        self._post(now + s_to_ns(ln.profile.latency_s), _DELIVERED, ch.payload_id, (link_idx, ch))
        self._pump(ln, now)

    def _chunk_delivered(self, link_idx: int, ch, now: int) -> None:
        ln = self._links[link_idx]
        self._note_link(ln, now, ch.payload_id, ch.index, ch.size_bytes, ch.phase_class, "deliver")
        if not ch.is_last:
            return
        mb = ln.owner.pop(ch.payload_id)
        payload = ln.payloads.pop(ch.payload_id)
        ln.sent_bytes.pop(ch.payload_id, None)
        self._note(now, EventKind.PAYLOAD_DELIVERED, ch.payload_id, ln.dst)
        self.backend.delivered(link_idx, payload, mb, now)
        if ln.is_return:
            self._emit_tokens(mb, now)
            self._want_boundary(now)
        else:
            dst = self._stages[ln.dst]
            dst.waiting.append(mb)
            self._launch_compute(dst, now)

    # --------------------------------------------------------------- head
    def _emit_tokens(self, mb, now: int) -> None:
        self._inflight.pop(mb.id, None)
        t_s = now / NS
        for rid in mb.request_ids:
            r = self._requests[rid]
            r.tokens_emitted += 1
            self._emissions.append((now, rid))
            if r.state is RequestState.PREFILL:
                r.first_token_time = t_s
                if r.output_len == 1:
                    r.state, r.finish_time = RequestState.FINISHED, t_s
                else:
                    r.state = RequestState.DECODING
                    self._ready.append(r)
            elif r.state is RequestState.DECODING:
                if r.tokens_emitted >= r.output_len:
                    r.state, r.finish_time = RequestState.FINISHED, t_s
                else:
                    self._ready.append(r)
        self.backend.feedback(mb, now)

    def _want_boundary(self, now: int) -> None:
        if now not in self._boundaries:
            self._boundaries.add(now)
            self._post(now, _BOUNDARY, self._iteration + 1)

    def _boundary(self, now: int) -> None:
        self._boundaries.discard(now)
        head = self._stages[0]
        if head.busy or head.waiting or not (self._ready or self._pending):
            return
        phase = Phase.DECODE if self._ready else Phase.PREFILL
        ctrl = self.cfg.controller
        if self._last_decision is None or self._iteration % ctrl.decision_stride == 0:
            decision = self._decide(phase)
        else:
            decision = self._last_decision
        room = decision.n_microbatches - len(self._inflight)
        if room <= 0:
            return
        batches = pipelink.admit_and_batch(
            self._ready, self._pending, decision, ctrl.max_batch_size, room, now / NS,
            allow_mixed=self.cfg.allow_mixed_phase, id_start=self._next_mb)
        if not batches:
            return
        self._iteration += 1
        self._last_decision = decision
        self._decisions.append((self._iteration, decision))
        self._note(now, EventKind.ITERATION_BOUNDARY, self._iteration, 0)
        self._next_mb += len(batches)
        for mb in batches:
            self._inflight[mb.id] = mb
            for rid in mb.request_ids:
                r = self._requests[rid]
                if r.state is RequestState.QUEUED:
                    r.state = RequestState.PREFILL
            head.waiting.append(mb)
            self.backend.admit(mb, now)
        self._launch_compute(head, now)

    # ---------------------------------------------------------------- run
    def _reset(self) -> None:
        policy = (T_.LinkPolicy.DECODE_PRIORITY
                  if self.cfg.scheduling_policy is E.SchedulingPolicy.DECODE_PRIORITY
                  else T_.LinkPolicy.FCFS)
        self._stages = [_StageState(i, p) for i, p in enumerate(self.stage_profiles)]
        nl = len(self.link_profiles)
        self._links = [
            _LinkState(i, lp, T_.LinkQueue(chunk_size=self.cfg.chunk_size, policy=policy),
                       0 if i == nl - 1 else i + 1, i == nl - 1)
            for i, lp in enumerate(self.link_profiles)
        ]
        self._heap, self._seq = [], 0
        self._requests, self._pending, self._ready = {}, deque(), deque()
        self._inflight: dict = {}
        self._boundaries: set = set()
        self._events, self._link_log, self._decisions, self._emissions = [], [], [], []
        self._first_compute: dict = {}
        self._iteration = self._next_mb = self._next_payload = 0
        self._last_decision = None

    def run(self, trace, horizon_s: float | None = None):
        self._reset()
        seen = set()
        for r in trace.requests:
            if r.id in seen:
                raise pipelink.ConfigError(f"duplicate request id {r.id} in trace")
            seen.add(r.id)
            req = r.fresh_copy()
            t = s_to_ns(r.arrival_time)
            req.arrival_time = t / NS
            self._requests[r.id] = req
            self._post(t, _ARRIVAL, r.id)
        self.backend.start(self, trace)
        horizon = None if horizon_s is None else s_to_ns(horizon_s)
        last = 0
        heap = self._heap
        while heap:
            if horizon is not None and heap[0][0] > horizon:
                last = horizon
                break
            t, kind, subject, _, data = heapq.heappop(heap)
            if t > last:
                last = t
            if kind == _DELIVERED:
                self._chunk_delivered(data[0], data[1], t)
            elif kind == _DONE:
                self._compute_finished(data, subject, t)
            elif kind == _ARRIVAL:
                self._pending.append(self._requests[subject])
                self._note(t, EventKind.ARRIVAL, subject)
                self._want_boundary(t)
            elif kind == _BOUNDARY:
                self._boundary(t)
            else:
                self._chunk_sent(data[0], data[1], t)
        for st in self._stages:
            if st.busy:
                st.intervals.append((st.started, last))
                st.busy = False
        reqs = [self._requests[k] for k in sorted(self._requests)]
        links = [e for _, e in sorted(enumerate(self._link_log), key=lambda p: (p[1].time_ns, p[0]))]
        result = E.RunResult(
            requests=reqs, events=self._events, link_events=links, decisions=self._decisions,
            stage_busy_ns=[st.intervals for st in self._stages], token_emissions=self._emissions,
            first_compute_ns=self._first_compute, end_ns=last,
            all_finished=all(r.state is RequestState.FINISHED for r in reqs))
        self.backend.finish(result)
        return result
