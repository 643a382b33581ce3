"""Backend hooks on the reference's own event loop (the Python twin of csrc/sched.cu).

``PipelineDriver`` subclasses the unmodified ``pipelink.PipelineEngine``
(pipelink/engine.py:264-600): the reference's ``run`` loop, heap tie order,
boundary rule, ``choose_n``, ``admit_and_batch``, ``LinkQueue`` and payload
sizing all execute unchanged, so the schedule, chunk boundaries and token
accounting *are* the reference's.  The subclass only observes four of the
engine's own methods and fires a backend hook at each simulated step, where
the B200 backend issues the real work:

  hook                      reference method (site)            B200 backend action
  ------------------------  ---------------------------------  ---------------------------------
  admit(mb)                 _on_boundary (E:481-504), seen     build KV block tables / metadata
                            at the head's first start
  compute(stage, mb)        _try_start_compute (E:376-388)     pl_stage_forward on the stage stream
  emit(link, chunk, off)    _link_emit_next (E:347-356)        one NCCL send/recv (or peer copy) of
                                                               bytes [off, off+size) of the payload
  feedback(mb)              _apply_feedback (E:422-442)        return hop landed: release the slot

``_link_emit_next`` gets at the chunk it put on the wire through the link's
queue: each link's ``LinkQueue`` is replaced (same chunk size and policy) by a
subclass that remembers the payloads it was given and the chunk it last
yielded -- ``LinkQueue``'s own ``enqueue``/``next_chunk`` still decide.
Decisions never depend on completions, so the returned ``RunResult`` is the
reference's own (tests/test_driver_parity.py) while the GPU executes the
resulting DAG asynchronously in per-stage FIFO order.
"""

from __future__ import annotations

from ._pipelink import pipelink

E = pipelink.engine
T_ = pipelink.transport


class Backend:
    """No-op hooks (pure virtual run).  Subclasses issue real work."""

    def start(self, driver: "PipelineDriver", trace) -> None: ...
    def admit(self, mb, now_ns: int) -> None: ...
    def compute(self, stage: int, mb, now_ns: int) -> None: ...
    def emit(self, link: int, payload, chunk, offset: int, now_ns: int) -> None: ...
    def feedback(self, mb, now_ns: int) -> None: ...
    def finish(self, result) -> None: ...


class _TapQueue(T_.LinkQueue):
    """The reference LinkQueue, recording what the engine enqueued and took."""

    def __init__(self, chunk_size, policy):
        super().__init__(chunk_size=chunk_size, policy=policy)
        self.payloads: dict = {}      # payload id -> Payload (until its last chunk leaves)
        self.offsets: dict = {}       # payload id -> bytes already chunked out
        self.taken = None             # (payload, chunk, offset) of the last next_chunk()

    def enqueue(self, payload) -> None:
        super().enqueue(payload)
        self.payloads[payload.id] = payload
        self.offsets[payload.id] = 0

    def next_chunk(self):
        ch = super().next_chunk()
        if ch is None:
            self.taken = None
            return None
        off = self.offsets[ch.payload_id]
        payload = self.payloads[ch.payload_id]
        if ch.is_last:
            del self.payloads[ch.payload_id], self.offsets[ch.payload_id]
        else:
            self.offsets[ch.payload_id] = off + ch.size_bytes
        self.taken = (payload, ch, off)
        return ch


class PipelineDriver(E.PipelineEngine):
    """``pipelink.PipelineEngine`` whose simulated compute and link steps also call a
    backend.  Same constructor, same ``run(trace, horizon_s)`` and ``RunResult``."""

    def __init__(self, cfg, cluster, stage_profiles, backend: Backend | None = None):
        super().__init__(cfg, cluster, stage_profiles)
        self.backend = backend or Backend()

    def set_link_profiles(self, link_profiles) -> None:
        """Swap in measured link estimates (forward hops + return hop, cluster order)."""
        if len(link_profiles) != len(self.link_profiles):
            raise pipelink.ConfigError("link profile count must equal the hop count")
        self.link_profiles = list(link_profiles)

    def set_stage_profiles(self, stage_profiles) -> None:
        """Swap in measured profiles (startup profiling) before the next run."""
        if len(stage_profiles) != len(self.stage_profiles):
            raise pipelink.ConfigError("profile count must equal the stage count")
        self.stage_profiles = list(stage_profiles)

    # ------------------------------------------------------------ hooks
    def _reset(self) -> None:
        super()._reset()
        for link in self._links:
            q = link.queue
            link.queue = _TapQueue(q.chunk_size, q.policy)
        self._admitted = -1           # highest micro-batch id handed to backend.admit

    def _try_start_compute(self, stage, now: int) -> None:
        was_busy = stage.busy
        super()._try_start_compute(stage, now)
        if was_busy or not stage.busy:
            return
        mb = stage.current
        if stage.idx == 0 and mb.id > self._admitted:
            # the boundary that admitted this micro-batch (and its siblings, queued behind
            # it on the head) starts the head at the same instant (E:505)
            for m in [mb, *stage.queue]:
                if m.id > self._admitted:
                    self.backend.admit(m, now)
                    self._admitted = m.id
        self.backend.compute(stage.idx, mb, now)

    def _link_emit_next(self, link, now: int) -> None:
        super()._link_emit_next(link, now)
        taken = link.queue.taken
        if taken is not None and link.busy:
            link.queue.taken = None
            payload, ch, off = taken
            self.backend.emit(link.idx, payload, ch, off, now)

    def _apply_feedback(self, mb, now: int) -> None:
        super()._apply_feedback(mb, now)
        self.backend.feedback(mb, now)

    def run(self, trace, horizon_s: float | None = None):
        self.backend.start(self, trace)
        result = super().run(trace, horizon_s)
        self.backend.finish(result)
        return result
