"""Live pipeline over NVLink with real B200 compute (one stage per rank, S >= 2).

Twin of the reference's ``run_socket_demo`` (pipelink/demo.py:52-196): the head
loop runs the unchanged ``choose_n`` + ``admit_and_batch`` on every step and
reacts to token feedback as it arrives on the wall clock (no virtual clock), so
the micro-batch composition is timing dependent exactly as in the reference
demo; what must match the virtual run is the token
accounting -- and here also the generated ids.  Differences from the socket
demo: each stage is a real decoder stage on its own GPU (one process per GPU,
``torch.distributed`` world of S; the socket demo has exactly two stages), the
links are ``DeviceLinkSender`` /
``DeviceLinkReceiver`` over NCCL, and the forward payload carries the
micro-batch metadata ahead of the bf16 residual stream (the socket demo
prefixes a 4-byte request count, demo.py:161-163).

    result = run_device_demo(cfg, cluster, stage_profiles, trace, decoder=TINY)
    result.tokens_by_request   # {rid: count}   (rank 0)
    result.tokens              # {rid: ids}     (rank 0)

Runtime monitoring: every stage writes the device-clock duration
of its last completed forward (phase, tokens, ms) into its slot of the frame header;
the tail returns all stages' reports after the token ids (the reference returns only
the 8-byte ids, demo.py:32-49).  The head feeds them, and each micro-batch's
dispatch-to-feedback time, to a ``RuntimeMonitor`` (monitor.py) that rebuilds the
StageProfiles / LinkProfiles ``choose_n`` plans with every ``monitor_epoch``
micro-batches (``monitor_epoch=0`` keeps the startup profiles).
"""

from __future__ import annotations

import ctypes as C
import queue
import time
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._pipelink import pipelink
from .backend import GpuBackend, Placement
from .wire import DeviceLinkReceiver, DeviceLinkSender

BatchPhase = pipelink.engine.BatchPhase
RequestState = pipelink.RequestState
PayloadClass = pipelink.PayloadClass
Phase = pipelink.Phase
HDR0 = 8  # int32 words: T, R, phase, max_seqlen, max_ctx, slot, meta_len, reserved
# then 3 words per stage: the stage's last completed forward (phase, tokens, ms as f32 bits)


def hdr_words(S: int) -> int:
    return HDR0 + 3 * S


class _FwdClock:
    """CUDA events around a stage's forwards; reports the latest completed one."""

    def __init__(self):
        self.q = deque()
        self.last = (0, 0, 0.0)

    def start(self, stream):
        a = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        return a

    def stop(self, a, stream, phase: int, T: int):
        b = torch.cuda.Event(enable_timing=True)
        b.record(stream)
        self.q.append((phase, T, a, b))

    def report(self) -> tuple[int, int, float]:
        while self.q and self.q[0][3].query():
            phase, T, a, b = self.q.popleft()
            self.last = (phase, T, a.elapsed_time(b))
        return self.last


def _report_words(rep) -> np.ndarray:
    return np.array([rep[0], rep[1], np.float32(rep[2]).view(np.int32)], dtype=np.int32)


@dataclass
class LiveResult:
    tokens_by_request: dict
    tokens: dict
    wall_s: float
    microbatches: int
    monitor_updates: int = 0
    stage_profiles: list | None = None   # the monitor's latest estimates
    link_profiles: list | None = None


class _Requests:
    """The `_requests` view GpuBackend.admit reads (driver stand-in)."""

    def __init__(self, reqs):
        self._requests = {r.id: r for r in reqs}


def _hop_comms(S: int) -> dict:
    """One 2-rank communicator per hop: forward hops s -> s+1 and the return hop
    S-1 -> 0 (the sender is comm-rank 0).  Returns {hop: handle} for this rank's hops;
    hop S-1 is the return hop."""
    import torch.distributed as dist

    me = dist.get_rank()
    hops = [(s, s + 1) for s in range(S - 1)] + [(S - 1, 0)]
    comms = {}
    for hop, (src, dst) in enumerate(hops):
        obj = [None]
        if me == src:
            buf = (C.c_uint8 * 128)()
            N.call("pl_nccl_unique_id", buf, 128)
            obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=src)
        if me in (src, dst):
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            h = C.c_void_p()
            N.call("pl_comm_init_rank", uid, 2, 0 if me == src else 1, C.byref(h))
            comms[hop] = h
    # Establish every P2P connection now, from one thread, in the same order on all
    # ranks: NCCL connects lazily on first use, and a connect issued while another
    # link's receive kernel spins on the same GPU can wait on that kernel forever.
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = torch.zeros(8, dtype=torch.int64, device=dev)
    st = torch.cuda.Stream(dev)
    for hop, (src, dst) in enumerate(hops):
        if me == src:
            N.call("pl_p2p_send", comms[hop], buf.data_ptr(), 64, 1, st.cuda_stream)
        elif me == dst:
            N.call("pl_p2p_recv", comms[hop], buf.data_ptr(), 64, 0, st.cuda_stream)
        st.synchronize()
        dist.barrier()
    return comms


def run_device_demo(cfg, cluster, stage_profiles, trace, *, decoder, seed: int = 0,
                    timeout_s: float = 120.0, monitor_epoch: int = 32) -> LiveResult | None:
    import torch.distributed as dist

    S = len(cfg.partition.stages)
    if S < 2 or not dist.is_initialized() or dist.get_world_size() != S:
        raise pipelink.ConfigError("the live demo runs one stage per rank (world size == stages >= 2)")
    rank = dist.get_rank()
    names = cfg.partition.node_names()
    link_profiles = [cluster.link(a, b) for a, b in list(zip(names, names[1:])) + [(names[-1], names[0])]]
    policy = (pipelink.LinkPolicy.DECODE_PRIORITY
              if cfg.scheduling_policy.value == "decode_priority" else pipelink.LinkPolicy.FCFS)
    bytes_per_token = cfg.model.hidden_dim * cfg.model.dtype_bytes
    placement = Placement(S, S, rank)
    be = GpuBackend(decoder, cfg, placement, seed=seed)
    requests = {r.id: r.fresh_copy() for r in trace.requests}
    view = _Requests(requests.values())
    be.start(view, trace)
    exe = be.exe[rank]
    dev = exe.device
    comms = _hop_comms(S)
    comm_ret = comms.get(S - 1)  # the return hop: tail and head only
    if rank == S - 1:
        _tail(be, exe, comms[S - 2], comm_ret, cfg, policy, timeout_s, S)
        return None
    if rank > 0:
        _middle(exe, comms[rank - 1], comms[rank], cfg, policy, timeout_s, S, rank)
        return None
    return _head(be, exe, comms[0], comm_ret, cfg, policy, requests, trace, stage_profiles,
                 link_profiles, bytes_per_token, timeout_s, dev, S, monitor_epoch)


def _tail(be, exe, comm_fwd, comm_ret, cfg, policy, timeout_s, S):
    # return link: this rank created it, so it is comm-rank 0 and the head is peer 1
    ret = DeviceLinkSender(comm_ret, 1, cfg.chunk_size, policy, "ret-sender", exe.device)
    ret.start()
    stream = exe.stream
    HDR = hdr_words(S)
    clock = _FwdClock()

    def on_payload(p):
        hdr = p.body[: HDR * 4].view(torch.int32).cpu().numpy()
        T, R, phase, max_seqlen, max_ctx, slot, meta_len = (int(x) for x in hdr[:7])
        meta_b = p.body[HDR * 4: HDR * 4 + meta_len * 4]
        hid_b = p.body[HDR * 4 + meta_len * 4:]
        with torch.cuda.stream(stream):
            stream.wait_stream(torch.cuda.current_stream())
            exe.meta_dev[:meta_len].view(torch.uint8).copy_(meta_b)
            exe.hidden[slot][:T].view(torch.uint8).reshape(-1).copy_(hid_b)
        a = clock.start(stream)
        exe.forward(slot, T, R, phase == 1, max_seqlen, max_ctx)
        clock.stop(a, stream, phase, T)
        # [ids | every stage's report]: the head's monitor reads the trailer
        reports = hdr[HDR0:HDR].copy()
        reports[3 * (S - 1): 3 * S] = _report_words(clock.report())
        trailer = torch.from_numpy(reports.view(np.int64) if reports.size % 2 == 0 else
                                   np.concatenate([reports, np.zeros(1, np.int32)]).view(np.int64))
        with torch.cuda.stream(stream):
            ids = torch.cat([exe.out_ids[slot][:R], trailer.to(exe.device, non_blocking=False)])
        ev = torch.cuda.Event()
        ev.record(stream)
        fb = pipelink.Payload(id=p.payload_id, phase_class=PayloadClass.DECODE,
                              size_bytes=ids.numel() * 8, micro_batch_id=p.payload_id, enqueue_time=0)
        ret.send(fb, ids, ready=ev)

    recv = DeviceLinkReceiver(comm_fwd, 0, on_payload, "tail-recv", exe.device)
    recv.run()  # inline: this thread is the tail stage (demo.py:32-49)
    ret.close()
    ret.join(timeout=timeout_s)
    if recv.failed:
        raise pipelink.ProtocolError(f"tail receiver failed: {recv.error!r}")


def _middle(exe, comm_in, comm_out, cfg, policy, timeout_s, S, rank):
    """A stage between head and tail: receive [header | metadata | residual stream],
    run the stage forward in place, pass the same framing on to the next rank."""
    nxt = DeviceLinkSender(comm_out, 1, cfg.chunk_size, policy, "mid-sender", exe.device)
    nxt.start()
    stream = exe.stream
    HDR = hdr_words(S)
    clock = _FwdClock()

    def on_payload(p):
        hdr = p.body[: HDR * 4].view(torch.int32).cpu().numpy()
        T, R, phase, max_seqlen, max_ctx, slot, meta_len = (int(x) for x in hdr[:7])
        off = HDR * 4 + meta_len * 4
        with torch.cuda.stream(stream):
            stream.wait_stream(torch.cuda.current_stream())
            exe.meta_dev[:meta_len].view(torch.uint8).copy_(p.body[HDR * 4: off])
            exe.hidden[slot][:T].view(torch.uint8).reshape(-1).copy_(p.body[off:])
        a = clock.start(stream)
        exe.forward(slot, T, R, phase == 1, max_seqlen, max_ctx)
        clock.stop(a, stream, phase, T)
        rep_w = torch.from_numpy(_report_words(clock.report()).view(np.uint8))
        with torch.cuda.stream(stream):
            p.body[off:].copy_(exe.hidden[slot][:T].view(torch.uint8).reshape(-1))  # reuse the frame
            o = (HDR0 + 3 * rank) * 4
            p.body[o: o + 12].copy_(rep_w.to(exe.device))
        ev = torch.cuda.Event()
        ev.record(stream)
        out = pipelink.Payload(id=p.payload_id, phase_class=p.phase_class, size_bytes=p.body.numel(),
                               micro_batch_id=p.payload_id, enqueue_time=0)
        nxt.send(out, p.body, ready=ev)

    recv = DeviceLinkReceiver(comm_in, 0, on_payload, "mid-recv", exe.device)
    recv.run()  # inline: this thread is the stage
    nxt.close()
    nxt.join(timeout=timeout_s)
    if recv.failed:
        raise pipelink.ProtocolError(f"stage receiver failed: {recv.error!r}")


def _head(be, exe, comm_fwd, comm_ret, cfg, policy, requests, trace, stage_profiles, link_profiles,
          bytes_per_token, timeout_s, dev, S, monitor_epoch):
    from .monitor import RuntimeMonitor

    monitor = RuntimeMonitor(stage_profiles, link_profiles, epoch=max(1, monitor_epoch))
    HDR = hdr_words(S)
    clock = _FwdClock()
    sent_at: dict = {}
    fwd = DeviceLinkSender(comm_fwd, 1, cfg.chunk_size, policy, "fwd-sender", dev)
    feedback: queue.Queue = queue.Queue()
    head_recv = DeviceLinkReceiver(comm_ret, 0, feedback.put, "head-recv", dev)  # tail = comm-rank 0
    fwd.start()
    head_recv.start()
    pending = deque(requests[r.id] for r in trace.requests)
    ready: deque = deque()
    in_flight: dict = {}
    payload_mb: dict = {}
    next_mb = next_payload = 0
    unfinished = len(requests)
    n_mbs = 0
    t0 = time.perf_counter()
    scatter_stream = torch.cuda.Stream(dev)

    def apply_feedback(p) -> int:
        nonlocal stage_profiles, link_profiles
        mb = payload_mb.pop(p.payload_id)
        in_flight.pop(mb.id)
        rec = be.mbs[mb.id]
        ids = p.body.view(torch.int64)[: rec.R]
        be._scatter(rec, ids, scatter_stream)
        if monitor_epoch > 0:
            rtt = time.perf_counter() - sent_at.pop(mb.id)
            with torch.cuda.stream(scatter_stream):  # never the legacy default stream
                words = p.body.view(torch.int64)[rec.R:].cpu().numpy().view(np.int32)[: 3 * S]
            compute = 0.0
            for s in range(S):
                ph, T, ms = int(words[3 * s]), int(words[3 * s + 1]), float(words[3 * s + 2:3 * s + 3].view(np.float32)[0])
                if T > 0:
                    monitor.stage_sample(s, Phase.DECODE if ph == 1 else Phase.PREFILL, T, ms / 1e3)
                    compute += ms / 1e3
            monitor.round_trip(rec.T * bytes_per_token, rtt, compute)
            if monitor.tick():
                stage_profiles, link_profiles = monitor.stage_profiles, monitor.link_profiles
        done = 0
        for rid in mb.request_ids:
            r = requests[rid]
            r.tokens_emitted += 1
            if r.state is RequestState.PREFILL:
                if r.output_len == 1:
                    r.state = RequestState.FINISHED
                    done += 1
                else:
                    r.state = RequestState.DECODING
                    ready.append(r)
            elif r.state is RequestState.DECODING:
                if r.tokens_emitted >= r.output_len:
                    r.state = RequestState.FINISHED
                    done += 1
                else:
                    ready.append(r)
        be.feedback(mb, 0)
        return done

    try:
        while unfinished > 0:
            dispatched = False
            if ready or pending:
                phase = Phase.DECODE if ready else Phase.PREFILL
                demand = len(ready) + sum(m.batched_tokens for m in in_flight.values()) + \
                    sum(r.input_len for r in pending)
                decision = pipelink.choose_n(cfg.controller, stage_profiles, link_profiles, demand, phase,
                                             bytes_per_token=bytes_per_token)
                room = decision.n_microbatches - len(in_flight)
                if room > 0:
                    batches = pipelink.admit_and_batch(ready, pending, decision, cfg.controller.max_batch_size,
                                                       room, now_s=0.0, allow_mixed=cfg.allow_mixed_phase,
                                                       id_start=next_mb)
                    next_mb += len(batches)
                    for mb in batches:
                        for rid in mb.request_ids:
                            if requests[rid].state is RequestState.QUEUED:
                                requests[rid].state = RequestState.PREFILL
                        in_flight[mb.id] = mb
                        be.admit(mb, 0)
                        a = clock.start(exe.stream)
                        be.compute(0, mb, 0)
                        rec = be.mbs[mb.id]
                        clock.stop(a, exe.stream, 1 if rec.decode else 0, rec.T)
                        body = _forward_body(exe, rec, dev, HDR, clock.report())
                        sent_at[mb.id] = time.perf_counter()
                        pclass = PayloadClass.DECODE if mb.phase is BatchPhase.DECODE else PayloadClass.PREFILL
                        payload = pipelink.Payload(id=next_payload, phase_class=pclass,
                                                   size_bytes=body.numel(), micro_batch_id=mb.id,
                                                   enqueue_time=0)
                        next_payload += 1
                        payload_mb[payload.id] = mb
                        fwd.send(payload, body)
                        dispatched = True
                        n_mbs += 1
            if not dispatched:
                if not in_flight:
                    raise pipelink.ProtocolError("demo stalled with no work in flight")
                unfinished -= apply_feedback(feedback.get(timeout=timeout_s))
    finally:
        fwd.close()
        fwd.join(timeout=timeout_s)
        head_recv.join(timeout=timeout_s)
    torch.cuda.synchronize(dev)
    gen = be.gen_tokens.cpu().numpy()
    toks = {rid: gen[be.rid_index[rid], : r.tokens_emitted].copy() for rid, r in requests.items()}
    return LiveResult(tokens_by_request={rid: requests[rid].tokens_emitted for rid in sorted(requests)},
                      tokens=toks, wall_s=time.perf_counter() - t0, microbatches=n_mbs,
                      monitor_updates=monitor.updates, stage_profiles=monitor.stage_profiles,
                      link_profiles=monitor.link_profiles)


def _forward_body(exe, rec, dev, HDR, report) -> torch.Tensor:
    """[int32 header (+ per-stage reports) | int32 metadata | bf16 residual stream] of one
    micro-batch (device); the head's own report goes into stage slot 0."""
    meta = rec.meta
    hdr = np.zeros(HDR, dtype=np.int32)
    hdr[:HDR0] = [rec.T, rec.R, 1 if rec.decode else 0, rec.max_seqlen, rec.max_ctx, rec.slot, meta.size, 0]
    hdr[HDR0:HDR0 + 3] = _report_words(report)
    prefix = np.concatenate([hdr, meta]).view(np.uint8)
    hid_bytes = rec.T * exe.spec.d * 2
    body = torch.empty(prefix.size + hid_bytes, dtype=torch.uint8, device=dev)
    st = exe.stream
    with torch.cuda.stream(st):
        body[: prefix.size].copy_(torch.from_numpy(prefix), non_blocking=False)
        body[prefix.size:].copy_(exe.hidden[rec.slot][: rec.T].view(torch.uint8).reshape(-1))
    ev = torch.cuda.Event()
    ev.record(st)
    ev.synchronize()
    return body
