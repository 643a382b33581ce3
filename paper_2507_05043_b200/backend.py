"""B200 backend for the virtual-clock driver: real stage forwards and real links.

Every rank runs the identical deterministic driver (decisions come from the
virtual clock, never from completions), so all ranks agree on the schedule
without exchanging control messages; each rank only issues the work of its
own stages and links.  Per local stage there are three CUDA streams:

  compute   H2D micro-batch metadata -> pl_stage_forward
  send      outgoing link: one NCCL send (or device copy) per LinkQueue chunk
  recv      incoming link: one NCCL recv per chunk into the same byte range

Cross-stream ordering uses CUDA events (never host syncs):
  compute(s, mb)   waits recv_done(s, slot) and the previous occupant's send_done(s, slot)
  send chunk       waits comp_done(s, slot) (first chunk)
  recv chunk       waits the previous occupant's send_done(dst, slot) (first chunk)
  head decode      waits the latest token-scatter event (return hop)
A micro-batch keeps one slot (= one hidden buffer per stage) from admission
until its tokens come back (engine.py:478 caps in-flight micro-batches at n).

Transports per hop: NCCL 2.28 ncclSend/ncclRecv between ranks
(one 2-rank communicator per directed hop, NVLink/NVSwitch), a device copy
when both stages live on the same process.
"""

from __future__ import annotations

import ctypes as C
import os
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._pipelink import pipelink
from .driver import Backend
from .executor import StageExecutor, build_meta
from .spec import BLOCK_SIZE, DecoderSpec, prompt_tokens

transmission_ns = pipelink.transport.transmission_ns
s_to_ns = pipelink.transport.s_to_ns

BatchPhase = pipelink.engine.BatchPhase
RequestState = pipelink.RequestState

RUN_AHEAD = 24  # max launched-but-unfinished forwards per stage before the host waits


@dataclass
class _MbRec:
    slot: int
    T: int
    R: int
    decode: bool
    max_seqlen: int
    max_ctx: int
    meta: np.ndarray
    ids: np.ndarray | None
    scatter: np.ndarray  # int32 [req_slot R | out_pos R]
    rids: tuple = ()
    n_decode: int = 0    # mixed batch: leading decode requests (rows [0, n_decode))


def local_device_index(default: int = 0) -> int:
    """This process's GPU: LOCAL_RANK (one process per GPU)."""
    return int(os.environ.get("LOCAL_RANK", default))


class Placement:
    """Stage -> (rank, device).  Contiguous blocks of stages per rank."""

    def __init__(self, n_stages: int, world_size: int = 1, rank: int = 0,
                 devices: list | None = None):
        if n_stages % world_size:
            raise pipelink.ConfigError(f"{n_stages} stages do not split over {world_size} ranks")
        self.n_stages, self.world, self.rank = n_stages, world_size, rank
        per = n_stages // world_size
        self.stage_rank = [s // per for s in range(n_stages)]
        if world_size > 1:
            local = local_device_index(rank)
            self.stage_device = [torch.device("cuda", local) if self.stage_rank[s] == rank else None
                                 for s in range(n_stages)]
        else:
            devs = devices or [torch.device("cuda", 0)]
            self.stage_device = [torch.device(devs[s * len(devs) // n_stages]) for s in range(n_stages)]

    def local(self, s: int) -> bool:
        return self.stage_rank[s] == self.rank


class _PinnedRing:
    """Pinned host staging buffers reused round-robin, each guarded by an event."""

    def __init__(self, n: int, nbytes: int, device):
        self.bufs = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(n)]
        self.events = [None] * n
        self.i = 0
        self.device = device

    def take(self) -> tuple[int, torch.Tensor]:
        k = self.i
        self.i = (self.i + 1) % len(self.bufs)
        ev = self.events[k]
        if ev is not None:
            ev.synchronize()
        return k, self.bufs[k]

    def mark(self, k: int, stream) -> None:
        ev = torch.cuda.Event()
        ev.record(stream)
        self.events[k] = ev


class GpuBackend(Backend):
    def __init__(self, spec: DecoderSpec, cfg, placement: Placement, *, seed: int = 0,
                 prompts: dict | None = None, comms: dict | None = None, throttle: bool = False):
        self.spec, self.cfg, self.pl = spec, cfg, placement
        self.seed = seed
        self.user_prompts = prompts
        self.comms = comms or {}
        self.throttle = throttle
        self.record_links = False   # per-chunk CUDA events -> realized link log (device clock)
        # native runtime: decode payloads between stages of this process are stored by the
        # producer's last residual epilogue straight into the next stage's buffer
        self.fuse_transport = False  # opt-in: measured slower across GPUs
        self.S = placement.n_stages
        self.layer_ranges = [rng for _, rng in cfg.partition.stages]
        self.n_slots = cfg.controller.effective_n_max(self.S)
        self.exe: dict[int, StageExecutor] = {}
        self._built_for = None

    # ------------------------------------------------------------ build
    def prepare(self, trace) -> None:
        """Allocate weights / KV / buffers sized for `trace` (idempotent per shape)."""
        reqs = trace.requests
        max_in = max(r.input_len for r in reqs)
        max_ctx = max(r.input_len + r.output_len for r in reqs)
        ctrl = self.cfg.controller
        max_tokens = max(min(ctrl.max_batched_tokens, sum(r.input_len for r in reqs)), max_in,
                         min(ctrl.max_batch_size, len(reqs)))
        max_reqs = max(1, min(len(reqs), max(ctrl.max_batch_size, 1)))
        # prefill micro-batches can carry more requests than max_batch_size? no: capped
        blocks = sum(-(-(r.input_len + r.output_len) // BLOCK_SIZE) for r in reqs)
        key = (max_tokens, max_reqs, max_ctx, blocks)
        if self._built_for is not None and all(a >= b for a, b in zip(self._built_for, key)):
            return
        self.close()
        self.max_tokens, self.max_reqs, self.max_ctx, self.num_blocks = key
        self.max_blocks = -(-max_ctx // BLOCK_SIZE)
        for s in range(self.S):
            if not self.pl.local(s):
                continue
            lo, hi = self.layer_ranges[s]
            self.exe[s] = StageExecutor(
                self.spec, s, (lo, hi), s == 0, s == self.S - 1, self.pl.stage_device[s],
                seed=self.seed, max_tokens=max_tokens, max_reqs=max_reqs, max_ctx=max_ctx,
                num_blocks=blocks, n_slots=self.n_slots)
        self._built_for = key
        self._streams_built = False

    def _build_streams(self) -> None:
        self.send_stream, self.recv_stream = {}, {}
        self.ev_comp, self.ev_send, self.ev_recv = {}, {}, {}
        self.meta_ring, self.ids_ring = {}, {}
        self.throttle_ev = {}
        for s, exe in self.exe.items():
            dev = exe.device
            with torch.cuda.device(dev):
                self.send_stream[s] = torch.cuda.Stream(dev)
                self.recv_stream[s] = torch.cuda.Stream(dev)
            self.ev_comp[s] = [None] * self.n_slots
            self.ev_send[s] = [None] * self.n_slots
            self.ev_recv[s] = [None] * self.n_slots
            self.meta_ring[s] = _PinnedRing(RUN_AHEAD + 8, exe.meta_dev.numel() * 4, dev)
            if exe.is_first:
                self.ids_ring[s] = _PinnedRing(RUN_AHEAD + 8, exe.max_tokens * 8, dev)
            self.throttle_ev[s] = deque()
        head = self.exe.get(0)
        if head is not None:
            dev = head.device
            n_req = self._n_requests
            self.last_token = torch.zeros(n_req, dtype=torch.int64, device=dev)
            self.gen_tokens = torch.zeros(n_req, self._max_out, dtype=torch.int64, device=dev)
            self.ids_recv = [torch.zeros(self.max_reqs, dtype=torch.int64, device=dev)
                             for _ in range(self.n_slots)]
            self.scatter_dev = [torch.zeros(2 * self.max_reqs, dtype=torch.int32, device=dev)
                                for _ in range(self.n_slots)]
            self.scatter_ring = _PinnedRing(RUN_AHEAD + 8, 8 * self.max_reqs, dev)
        self._streams_built = True

    def close(self) -> None:
        self._native_close()
        for exe in self.exe.values():
            exe.close()
        self.exe = {}
        self._built_for = None

    # ------------------------------------------------------------ driver hooks
    def start(self, driver, trace) -> None:
        self.driver = driver
        self.prepare(trace)
        reqs = trace.requests
        self._n_requests = len(reqs)
        self._max_out = max(r.output_len for r in reqs)
        self.rid_index = {r.id: i for i, r in enumerate(reqs)}
        self._build_streams()
        self.req_len = {r.id: r.input_len for r in reqs}
        self.req_out = {r.id: r.output_len for r in reqs}
        self.free_slots = list(range(self.n_slots - 1, -1, -1))
        self.free_blocks = list(range(self.num_blocks - 1, -1, -1))
        self.bt_rows: dict[int, np.ndarray] = {}
        self.mbs: dict[int, _MbRec] = {}
        self.fb_events: list = []   # (event, mb request ids)
        self.mb_log: list = []      # (phase, R, sum of contexts) per admitted micro-batch
        self.first_decode_ev = None
        self.busy_events: list = []  # (stage, mb id, start event, end event) on the device clock
        self.chunk_events: list = []  # realized link log (record_links)
        self.mb_requests: dict = {}  # mb id -> request ids
        self.prompts = {}
        for r in reqs:
            if self.user_prompts is not None and r.id in self.user_prompts:
                p = np.asarray(self.user_prompts[r.id], dtype=np.int64)
                if p.shape != (r.input_len,):
                    raise pipelink.ConfigError(f"prompt of request {r.id} has wrong length")
            else:
                p = prompt_tokens(self.seed, r.id, r.input_len, self.spec.vocab)
            self.prompts[r.id] = p
        # t0 on every local device
        self.t0 = {}
        for s, exe in self.exe.items():
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(exe.stream)
            self.t0[s] = ev
        if self.throttle:
            self._start_gates()

    def admit(self, mb, now_ns: int) -> None:
        self.mb_requests[mb.id] = mb.request_ids
        slot = self.free_slots.pop()
        R = len(mb.request_ids)
        decode = mb.phase is BatchPhase.DECODE
        reqs = [self.driver._requests[rid] for rid in mb.request_ids]
        rows = np.empty((R, self.max_blocks), dtype=np.int32)
        for i, r in enumerate(reqs):
            bt = self.bt_rows.get(r.id)
            if bt is None:
                need = -(-(r.input_len + r.output_len) // BLOCK_SIZE)
                if len(self.free_blocks) < need:
                    raise pipelink.ConfigError("paged KV cache exhausted")
                bt = np.zeros(self.max_blocks, dtype=np.int32)
                bt[:need] = [self.free_blocks.pop() for _ in range(need)]
                self.bt_rows[r.id] = bt
            rows[i] = bt
        ridx = np.array([self.rid_index[r.id] for r in reqs], dtype=np.int32)
        out_pos = np.array([r.tokens_emitted for r in reqs], dtype=np.int32)
        if decode:
            T = R
            pos = np.array([r.input_len + r.tokens_emitted - 1 for r in reqs], dtype=np.int64)
            slots = rows[np.arange(R), pos // BLOCK_SIZE].astype(np.int64) * BLOCK_SIZE + pos % BLOCK_SIZE
            cu = np.arange(R + 1, dtype=np.int32)
            ctx = pos + 1
            last = np.arange(R, dtype=np.int32)
            meta = build_meta(T, R, self.max_blocks, pos, slots, ridx, cu, ctx, last, rows)
            rec = _MbRec(slot, T, R, True, 1, int(ctx.max()), meta, None,
                         np.concatenate([ridx, out_pos]).astype(np.int32), mb.request_ids)
            self.mb_log.append(("decode", R, int(ctx.sum())))
        elif mb.phase is BatchPhase.MIXED:
            # admit_and_batch places decoders ahead of prompts (engine.py:184-198)
            nd = 0
            while nd < R and reqs[nd].state is RequestState.DECODING:
                nd += 1
            if nd == 0 or any(r.state is RequestState.DECODING for r in reqs[nd:]):
                raise pipelink.ProtocolError("mixed micro-batch must lead with its decoders")
            dpos = np.array([r.input_len + r.tokens_emitted - 1 for r in reqs[:nd]], dtype=np.int64)
            plens = np.array([r.input_len for r in reqs[nd:]], dtype=np.int64)
            lens = np.concatenate([np.ones(nd, dtype=np.int64), plens])
            T = int(lens.sum())
            cu = np.zeros(R + 1, dtype=np.int64)
            np.cumsum(lens, out=cu[1:])
            ppos = np.arange(int(plens.sum()), dtype=np.int64) - np.repeat(cu[nd:-1] - nd, plens)
            pos = np.concatenate([dpos, ppos])
            req_of = np.repeat(np.arange(R), lens)
            slots = rows[req_of, pos // BLOCK_SIZE].astype(np.int64) * BLOCK_SIZE + pos % BLOCK_SIZE
            ctx = np.concatenate([dpos + 1, plens])
            meta = build_meta(T, R, self.max_blocks, pos, slots, np.repeat(ridx, lens), cu, ctx,
                              cu[1:] - 1, rows)
            ids = np.concatenate([np.zeros(nd, dtype=np.int64)] + [self.prompts[r.id] for r in reqs[nd:]])
            rec = _MbRec(slot, T, R, False, int(plens.max()), int((dpos + 1).max()), meta, ids,
                         np.concatenate([ridx, out_pos]).astype(np.int32), mb.request_ids, n_decode=nd)
            self.mb_log.append(("mixed", R, T))
        else:
            lens = np.array([r.input_len for r in reqs], dtype=np.int64)
            T = int(lens.sum())
            cu = np.zeros(R + 1, dtype=np.int64)
            np.cumsum(lens, out=cu[1:])
            pos = np.arange(T, dtype=np.int64) - np.repeat(cu[:-1], lens)
            req_of = np.repeat(np.arange(R), lens)
            slots = rows[req_of, pos // BLOCK_SIZE].astype(np.int64) * BLOCK_SIZE + pos % BLOCK_SIZE
            meta = build_meta(T, R, self.max_blocks, pos, slots, np.repeat(ridx, lens), cu, lens,
                              cu[1:] - 1, rows)
            ids = np.concatenate([self.prompts[r.id] for r in reqs])
            rec = _MbRec(slot, T, R, False, int(lens.max()), int(lens.max()), meta, ids,
                         np.concatenate([ridx, out_pos]).astype(np.int32), mb.request_ids)
            self.mb_log.append(("prefill", R, T))
        self.mbs[mb.id] = rec

    def compute(self, s: int, mb, now_ns: int) -> None:
        exe = self.exe.get(s)
        if exe is None:
            return
        rec = self.mbs[mb.id]
        st = exe.stream
        # run-ahead cap (also guards the pinned staging rings)
        q = self.throttle_ev[s]
        if len(q) >= RUN_AHEAD:
            q.popleft().synchronize()
        k = rec.slot
        if self.ev_send[s][k] is not None:
            st.wait_event(self.ev_send[s][k])
        if s > 0 and self.ev_recv[s][k] is not None:
            st.wait_event(self.ev_recv[s][k])
        if s == 0 and (rec.decode or rec.n_decode) and self.fb_events:
            st.wait_event(self.fb_events[-1][0])
            if self.first_decode_ev is None:
                self.first_decode_ev = torch.cuda.Event(enable_timing=True)
                self.first_decode_ev.record(st)
        lib = N.lib()
        i, buf = self.meta_ring[s].take()
        nb = rec.meta.nbytes
        buf[:nb].numpy()[:] = rec.meta.view(np.uint8)
        lib.pl_memcpy_async(exe.meta_dev.data_ptr(), buf.data_ptr(), nb, st.cuda_stream)
        self.meta_ring[s].mark(i, st)
        if s == 0 and not rec.decode:
            j, ib = self.ids_ring[s].take()
            ib[: rec.ids.nbytes].numpy()[:] = rec.ids.view(np.uint8)
            lib.pl_memcpy_async(exe.ids_dev.data_ptr(), ib.data_ptr(), rec.ids.nbytes, st.cuda_stream)
            self.ids_ring[s].mark(j, st)
        t_start = torch.cuda.Event(enable_timing=True)
        t_start.record(st)
        exe.forward(k, rec.T, rec.R, rec.decode, rec.max_seqlen, rec.max_ctx,
                    last_token=self.last_token if (s == 0) else None, n_decode=rec.n_decode)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(st)
        self.busy_events.append((s, mb.id, t_start, ev))  # ev also marks the payload's enqueue
        self.ev_comp[s][k] = ev
        q.append(ev)
        if self.S == 1:
            self._scatter(rec, exe.out_ids[k], st)

    def emit(self, link: int, payload, chunk, offset: int, now_ns: int) -> None:
        mb_id = payload.micro_batch_id
        rec = self.mbs[mb_id]
        k = rec.slot
        is_ret = link == self.S - 1
        src = self.S - 1 if is_ret else link
        dst = 0 if is_ret else link + 1
        src_local, dst_local = self.pl.local(src), self.pl.local(dst)
        first = offset == 0
        last = chunk.is_last
        size = chunk.size_bytes
        if src_local:
            sst = self.send_stream[src]
            if first:
                sst.wait_event(self.ev_comp[src][k])
            sbuf = (self.exe[src].out_ids[k] if is_ret else self.exe[src].hidden[k]).data_ptr() + offset
        if dst_local:
            dbuf = (self.ids_recv[k] if is_ret else self.exe[dst].hidden[k]).data_ptr() + offset
            prev_send = self.ev_send[dst][k]
        if src_local and self.record_links:
            t_emit = torch.cuda.Event(enable_timing=True)
        if src_local and dst_local:
            # same process: device (or peer) copy on the source's send stream
            if first and prev_send is not None:
                sst.wait_event(prev_send)
            if self.record_links:
                t_emit.record(sst)
            N.check(N.lib().pl_memcpy_async(dbuf, sbuf, size, sst.cuda_stream), "pl_memcpy_async")
            if self.record_links:
                self._note_chunk(link, src, k, payload, chunk, t_emit, sst)
            if last:
                ev = torch.cuda.Event()
                ev.record(sst)
                self.ev_send[src][k] = ev
                self._recv_done(dst, rec, ev, is_ret, self._deliver_ns(link, size, now_ns))
            return
        if src_local:
            comm = self.comms[link]
            if self.record_links:
                t_emit.record(sst)
            N.check(N.lib().pl_p2p_send(comm, sbuf, size, 1, sst.cuda_stream), "pl_p2p_send")
            if self.record_links:
                self._note_chunk(link, src, k, payload, chunk, t_emit, sst)
            if last:
                ev = torch.cuda.Event()
                ev.record(sst)
                self.ev_send[src][k] = ev
        if dst_local:
            rst = self.recv_stream[dst]
            if first and prev_send is not None:
                rst.wait_event(prev_send)
            comm = self.comms[link]
            N.check(N.lib().pl_p2p_recv(comm, dbuf, size, 0, rst.cuda_stream), "pl_p2p_recv")
            if last:
                ev = torch.cuda.Event()
                ev.record(rst)
                self._recv_done(dst, rec, ev, is_ret, self._deliver_ns(link, size, now_ns))

    def _note_chunk(self, link, src, slot, payload, chunk, t_emit, stream) -> None:
        t_sent = torch.cuda.Event(enable_timing=True)
        t_sent.record(stream)
        self.chunk_events.append((link, src, payload.id, chunk.index, chunk.size_bytes,
                                  chunk.phase_class, self.ev_comp[src][slot], t_emit, t_sent))

    def _deliver_ns(self, link: int, size: int, emit_ns: int) -> int:
        """Virtual delivery time of a chunk emitted at emit_ns (engine.py:355, 552-557)."""
        lp = self.driver.link_profiles[link]
        return emit_ns + transmission_ns(lp, size) + s_to_ns(lp.latency_s)

    def _recv_done(self, dst: int, rec: _MbRec, ev, is_ret: bool, deliver_ns: int) -> None:
        if self.throttle:
            # link-throttle mode: the payload becomes usable on the destination only once
            # the emulated link would have delivered it -- gated on a separate stream so the
            # link's own chunk pipeline is never held back by the latency
            ds = self.deliver_stream[dst]
            ds.wait_event(ev)
            N.check(N.lib().pl_gate_until_ns(self.t0_dev[dst].data_ptr(), deliver_ns, ds.cuda_stream),
                    "pl_gate_until_ns")
            ev = torch.cuda.Event()
            ev.record(ds)
        if not is_ret:
            self.ev_recv[dst][rec.slot] = ev
            return
        rst = self.recv_stream[0]
        rst.wait_event(ev)
        self._scatter(rec, self.ids_recv[rec.slot], rst)

    def _scatter(self, rec: _MbRec, ids: torch.Tensor, stream) -> None:
        """Return hop landed on the head: last_token / gen_tokens <- ids."""
        i, buf = self.scatter_ring.take()
        nb = rec.scatter.nbytes
        buf[:nb].numpy()[:] = rec.scatter.view(np.uint8)
        dev = self.scatter_dev[rec.slot]
        lib = N.lib()
        lib.pl_memcpy_async(dev.data_ptr(), buf.data_ptr(), nb, stream.cuda_stream)
        self.scatter_ring.mark(i, stream)
        R = rec.R
        N.check(lib.pl_token_scatter(ids.data_ptr(), dev.data_ptr(), dev.data_ptr() + 4 * R, R,
                                     self.last_token.data_ptr(), self.gen_tokens.data_ptr(),
                                     self.gen_tokens.stride(0), stream.cuda_stream), "pl_token_scatter")
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self.fb_events.append((ev, rec.rids))

    def feedback(self, mb, now_ns: int) -> None:
        rec = self.mbs.pop(mb.id)
        self.free_slots.append(rec.slot)
        for rid in mb.request_ids:
            r = self.driver._requests[rid]
            if r.state is RequestState.FINISHED:
                bt = self.bt_rows.pop(rid, None)
                if bt is not None:
                    need = -(-(r.input_len + r.output_len) // BLOCK_SIZE)
                    self.free_blocks.extend(int(b) for b in bt[:need][::-1])

    def finish(self, result) -> None:
        """Join all local streams, stop the clock, collect tokens and real timings."""
        self.timing = {}
        ends = {}
        for s, exe in self.exe.items():
            extra = (self.deliver_stream[s],) if self.throttle else ()
            for st in (self.send_stream[s], self.recv_stream[s], *extra):
                ev = torch.cuda.Event()
                ev.record(st)
                exe.stream.wait_event(ev)
            end = torch.cuda.Event(enable_timing=True)
            end.record(exe.stream)
            ends[s] = end
        for s, exe in self.exe.items():
            ends[s].synchronize()
        self.run_time_s = max((self.t0[s].elapsed_time(ends[s]) / 1e3 for s in self.exe), default=0.0)
        self.tokens = None
        self.fb_times_s, self.decode_start_s = [], None
        if 0 in self.exe:
            gen = self.gen_tokens.cpu().numpy()
            self.tokens = {r.id: gen[self.rid_index[r.id], : r.tokens_emitted].copy()
                           for r in result.requests}
            t0 = self.t0[0]
            self.fb_times_s = [t0.elapsed_time(ev) / 1e3 for ev, _ in self.fb_events]
        # realized link log on the source device's clock: enqueue = producing forward done,
        # emit/sent = the chunk's copy or ncclSend start/end on the link stream
        self.realized_links = []
        LinkEvent = pipelink.transport.LinkEvent
        seen = set()
        for link, src, pid, idx, size, pclass, ev_enq, ev_a, ev_b in self.chunk_events:
            t0s = self.t0[src]
            name = self.driver.link_profiles[link].name
            if (link, pid) not in seen:
                seen.add((link, pid))
                self.realized_links.append(LinkEvent(round(t0s.elapsed_time(ev_enq) * 1e6), name, pid, -1,
                                                     0, pclass, "enqueue"))
            ta, tb = round(t0s.elapsed_time(ev_a) * 1e6), round(t0s.elapsed_time(ev_b) * 1e6)
            self.realized_links.append(LinkEvent(ta, name, pid, idx, size, pclass, "emit"))
            self.realized_links.append(LinkEvent(tb, name, pid, idx, size, pclass, "sent"))
        # real per-stage busy intervals (ns on each device's clock, origin = run start)
        self.busy_real_ns = {}
        for s, mb_id, a, b in self.busy_events:
            t0s = self.t0[s]
            self.busy_real_ns.setdefault(s, []).append(
                (mb_id, round(t0s.elapsed_time(a) * 1e6), round(t0s.elapsed_time(b) * 1e6)))
            self.decode_start_s = (t0.elapsed_time(self.first_decode_ev) / 1e3
                                   if self.first_decode_ev is not None else None)

    # ------------------------------------------------------- native runtime
    def native_start(self, trace, record_links: bool = False):
        """Buffers + the native runtime (csrc/runtime.cu) for `trace`; returns the
        pl_pipeline handle that NativeScheduler.run drives.  The C++ twin of
        start/admit/compute/emit/feedback above: identical stream/event protocol,
        no Python on the per-micro-batch path."""
        self.prepare(trace)
        reqs = trace.requests
        self._n_requests = len(reqs)
        self._max_out = max(r.output_len for r in reqs)
        self.rid_index = {r.id: i for i, r in enumerate(reqs)}
        head = self.exe.get(0)
        if head is not None:
            with torch.cuda.device(head.device):
                self.last_token = torch.zeros(self._n_requests, dtype=torch.int64, device=head.device)
                self.gen_tokens = torch.zeros(self._n_requests, self._max_out, dtype=torch.int64,
                                              device=head.device)
        off = np.zeros(len(reqs) + 1, dtype=np.int64)
        parts = []
        for i, r in enumerate(reqs):
            if self.user_prompts is not None and r.id in self.user_prompts:
                p = np.asarray(self.user_prompts[r.id], dtype=np.int64)
                if p.shape != (r.input_len,):
                    raise pipelink.ConfigError(f"prompt of request {r.id} has wrong length")
            else:
                p = prompt_tokens(self.seed, r.id, r.input_len, self.spec.vocab)
            parts.append(p)
            off[i + 1] = off[i] + r.input_len
        ids = np.ascontiguousarray(np.concatenate(parts)) if parts else np.zeros(1, dtype=np.int64)
        h = self._native_handle(record_links)
        lt = self.last_token.data_ptr() if head is not None else None
        gen = self.gen_tokens.data_ptr() if head is not None else None
        stride = self.gen_tokens.stride(0) if head is not None else 1
        N.check(N.lib().pl_pipeline_set_requests(h, len(reqs), off.ctypes.data, ids.ctypes.data, lt, gen,
                                                 stride), "pl_pipeline_set_requests")
        self._native_record = record_links
        return h

    def _native_handle(self, record_links: bool):
        key = (self._built_for, bool(record_links), bool(self.throttle), bool(self.fuse_transport))
        if getattr(self, "_native", None) is not None and self._native[0] == key:
            return self._native[1]
        self._native_close()
        S, K = self.S, self.n_slots
        arr = lambda n: (C.c_void_p * max(1, n))()  # noqa: E731
        stage, stream, meta, ids, hidden, out_ids, comm = (arr(S), arr(S), arr(S), arr(S), arr(S * K),
                                                           arr(S * K), arr(S))
        dev = (C.c_int32 * S)()
        keep = []
        for s, exe in self.exe.items():
            stage[s] = exe.handle.value
            stream[s] = exe.stream.cuda_stream
            dev[s] = exe.device.index if exe.device.index is not None else 0
            meta[s] = exe.meta_dev.data_ptr()
            ids[s] = exe.ids_dev.data_ptr() if exe.ids_dev is not None else None
            for k in range(K):
                hidden[s * K + k] = exe.hidden[k].data_ptr()
                if exe.is_last:
                    out_ids[s * K + k] = exe.out_ids[k].data_ptr()
        for link, h in self.comms.items():
            comm[link] = h.value if isinstance(h, C.c_void_p) else h
        ids_recv = arr(K)
        head = self.exe.get(0)
        if head is not None:
            with torch.cuda.device(head.device):
                self._native_ids_recv = [torch.zeros(self.max_reqs, dtype=torch.int64, device=head.device)
                                         for _ in range(K)]
            for k, t in enumerate(self._native_ids_recv):
                ids_recv[k] = t.data_ptr()
        c = N.PipelineConfig()
        c.n_stages, c.n_slots, c.max_blocks, c.block_size = S, K, self.max_blocks, BLOCK_SIZE
        c.num_blocks, c.max_tokens, c.max_reqs, c.d = self.num_blocks, self.max_tokens, self.max_reqs, self.spec.d
        c.throttle, c.record_links = int(self.throttle), int(record_links)
        c.fuse_transport = int(self.fuse_transport)
        c.stage, c.stream, c.device = C.cast(stage, C.c_void_p), C.cast(stream, C.c_void_p), C.cast(dev, C.c_void_p)
        c.meta_dev, c.ids_dev = C.cast(meta, C.c_void_p), C.cast(ids, C.c_void_p)
        c.hidden, c.out_ids = C.cast(hidden, C.c_void_p), C.cast(out_ids, C.c_void_p)
        c.comm, c.ids_recv = C.cast(comm, C.c_void_p), C.cast(ids_recv, C.c_void_p)
        keep += [stage, stream, dev, meta, ids, hidden, out_ids, comm, ids_recv]
        h = C.c_void_p()
        N.check(N.lib().pl_pipeline_create(C.byref(c), C.byref(h)), "pl_pipeline_create")
        self._native = (key, h, keep)
        return h

    def _native_close(self) -> None:
        nat = getattr(self, "_native", None)
        if nat is not None:
            N.lib().pl_pipeline_destroy(nat[1])
            self._native = None

    def native_finish(self, result) -> None:
        """Device-clock results of the native run, in the attributes finish() sets."""
        lib = N.lib()
        h = self._native[1]
        cnt = np.zeros(5, dtype=np.int64)
        N.check(lib.pl_pipeline_counts(h, cnt.ctypes.data), "pl_pipeline_counts")
        nb, nf, nc, nm, nr = (int(x) for x in cnt)
        busy = np.zeros((nb, 2), dtype=np.int64)
        busy_s = np.zeros((nb, 2), dtype=np.float64)
        fb_mb = np.zeros(nf, dtype=np.int64)
        fb_s = np.zeros(nf, dtype=np.float64)
        ch = np.zeros((nc, 6), dtype=np.int64)
        ch_s = np.zeros((nc, 3), dtype=np.float64)
        mbl = np.zeros((nm, 4), dtype=np.int64)
        mb_off = np.zeros(nm + 1, dtype=np.int64)
        mb_ids = np.zeros(max(nr, 1), dtype=np.int64)
        rt, ds = C.c_double(), C.c_double()
        p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
        N.check(lib.pl_pipeline_read(h, C.byref(rt), C.byref(ds), p(busy), p(busy_s), p(fb_mb), p(fb_s), p(ch),
                                     p(ch_s), p(mbl), p(mb_off), p(mb_ids)), "pl_pipeline_read")
        self.run_time_s = rt.value
        self.decode_start_s = None if np.isnan(ds.value) else ds.value
        self.mb_requests = {int(m): tuple(mb_ids[mb_off[i]:mb_off[i + 1]].tolist())
                            for i, m in enumerate(mbl[:, 0].tolist())}
        self.mb_log = [(("prefill", "decode", "mixed")[d], int(R), int(w)) for _, d, R, w in mbl.tolist()]
        self.busy_real_ns = {}
        for (s, mb), (a, b) in zip(busy.tolist(), busy_s.tolist()):
            self.busy_real_ns.setdefault(s, []).append((mb, round(a * 1e9), round(b * 1e9)))
        self.fb_times_s = fb_s.tolist()
        self.fb_events = [(None, self.mb_requests.get(m, ())) for m in fb_mb.tolist()]
        self.tokens = None
        if 0 in self.exe:
            gen = self.gen_tokens.cpu().numpy()
            self.tokens = {r.id: gen[self.rid_index[r.id], : r.tokens_emitted].copy() for r in result.requests}
        self.realized_links = []
        if self._native_record:
            LinkEvent = pipelink.transport.LinkEvent
            classes = (pipelink.PayloadClass.PREFILL, pipelink.PayloadClass.DECODE)
            names = [lp.name for lp in self.driver.link_profiles]
            seen = set()
            for (link, _src, pid, idx, size, cls), (te, ta, tb) in zip(ch.tolist(), ch_s.tolist()):
                pclass = classes[cls]
                if (link, pid) not in seen:
                    seen.add((link, pid))
                    self.realized_links.append(LinkEvent(round(te * 1e9), names[link], pid, -1, 0, pclass,
                                                         "enqueue"))
                self.realized_links.append(LinkEvent(round(ta * 1e9), names[link], pid, idx, size, pclass, "emit"))
                self.realized_links.append(LinkEvent(round(tb * 1e9), names[link], pid, idx, size, pclass, "sent"))

    # ---------------------------------------------------------- throttle
    def _start_gates(self) -> None:
        """Per-device time origin on the GPU clock (%globaltimer) for the link gates."""
        self.t0_dev, self.deliver_stream = {}, {}
        for s, exe in self.exe.items():
            with torch.cuda.device(exe.device):
                self.deliver_stream[s] = torch.cuda.Stream(exe.device)
                t0 = torch.zeros(1, dtype=torch.int64, device=exe.device)
            N.check(N.lib().pl_record_globaltimer(t0.data_ptr(), exe.stream.cuda_stream),
                    "pl_record_globaltimer")
            ev = torch.cuda.Event()
            ev.record(exe.stream)
            self.deliver_stream[s].wait_event(ev)
            self.t0_dev[s] = t0
