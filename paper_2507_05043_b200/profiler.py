"""Startup profiling: measure ``StageProfile`` tables on the B200s.

The reference's compute model is a measured latency table per stage
(profiles.py:25-72; "startup profiling") that it never measures.
Here each stage times its own ``pl_stage_forward`` with CUDA events at a set
of token counts per phase; the tables feed the unchanged controller
(``choose_n``) and the virtual clock that drives the schedule.  Under
torchrun every rank profiles its stages and the tables are all-gathered, so
every rank runs the identical schedule.
"""

from __future__ import annotations

import numpy as np
import torch

from ._pipelink import pipelink
from .executor import StageExecutor, build_meta
from .spec import BLOCK_SIZE

Phase = pipelink.Phase

DECODE_POINTS = (1, 8, 16, 32, 64, 128, 256)
PREFILL_POINTS = (64, 512, 2048, 8192, 32768)


def _meta_for(exe: StageExecutor, T: int, decode: bool, ctx: int):
    if decode:
        R = T
        nb = -(-ctx // BLOCK_SIZE)
        rows = (np.arange(R * exe.max_blocks, dtype=np.int64) % max(1, exe.num_blocks)).reshape(R, -1)
        rows = rows.astype(np.int32)
        pos = np.full(R, ctx - 1, dtype=np.int64)
        slots = rows[np.arange(R), pos // BLOCK_SIZE].astype(np.int64) * BLOCK_SIZE + pos % BLOCK_SIZE
        meta = build_meta(T, R, exe.max_blocks, pos, slots, np.zeros(R), np.arange(R + 1),
                          pos + 1, np.arange(R), rows)
        del nb
        return meta, R, 1, ctx
    L = min(T, 512, exe.max_blocks * BLOCK_SIZE)  # prompts must fit the stage's block tables
    R = -(-T // L)  # prompts of L tokens, the last one shorter
    lens = np.full(R, L, dtype=np.int64)
    lens[-1] = T - L * (R - 1)
    cu = np.concatenate([[0], np.cumsum(lens)])
    pos = np.arange(T) - np.repeat(cu[:-1], lens)
    rows = (np.arange(R * exe.max_blocks, dtype=np.int64) % max(1, exe.num_blocks)).reshape(R, -1)
    rows = rows.astype(np.int32)
    req_of = np.repeat(np.arange(R), lens)
    slots = rows[req_of, pos // BLOCK_SIZE].astype(np.int64) * BLOCK_SIZE + pos % BLOCK_SIZE
    meta = build_meta(T, R, exe.max_blocks, pos, slots, np.zeros(T), cu, lens, cu[1:] - 1, rows)
    return meta, R, int(lens.max()), int(lens.max())


def time_forward(exe: StageExecutor, T: int, decode: bool, ctx: int = 512, reps: int = 3,
                 last_token: torch.Tensor | None = None) -> float:
    """Median device seconds of one stage forward at T tokens (weights streamed cold-ish)."""
    meta, R, max_seqlen, max_ctx = _meta_for(exe, T, decode, min(ctx, exe.max_ctx))
    if T > exe.max_tokens or R > exe.max_reqs:
        raise pipelink.ConfigError(f"profile point T={T} exceeds stage capacity")
    st = exe.stream
    with torch.cuda.stream(st):
        exe.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
        if exe.is_first:
            exe.ids_dev[:T].zero_()
        lt = last_token
        if exe.is_first and decode and lt is None:
            lt = torch.zeros(max(R, 1), dtype=torch.int64, device=exe.device)
    times = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        exe.forward(0, T, R, decode, max_seqlen, max_ctx, last_token=lt)
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    return float(np.median(times[1:]))


def profile_stage(exe: StageExecutor, decode_points=DECODE_POINTS, prefill_points=PREFILL_POINTS,
                  ctx: int = 512) -> pipelink.StageProfile:
    entries = {}
    for T in decode_points:
        if T <= min(exe.max_reqs, exe.max_tokens):
            entries[(Phase.DECODE, T)] = round(time_forward(exe, T, True, ctx), 7)
    for T in prefill_points:
        L = min(T, 512, exe.max_blocks * BLOCK_SIZE)
        if T <= exe.max_tokens and -(-T // L) <= exe.max_reqs:
            entries[(Phase.PREFILL, T)] = round(time_forward(exe, T, False, ctx), 7)
    # the reference requires >= 2 monotone points per phase (profiles.py:38-64)
    for ph in (Phase.DECODE, Phase.PREFILL):
        pts = sorted((t, s) for (p, t), s in entries.items() if p is ph)
        fixed, prev = [], 0.0
        for t, s in pts:
            prev = max(prev, s)
            fixed.append((t, prev))
        if len(fixed) == 1:
            t, s = fixed[0]
            fixed.append((t * 2, s * 2))
        for t, s in fixed:
            entries[(ph, t)] = s
    return pipelink.StageProfile(stage_id=exe.stage_idx, layers=exe.hi - exe.lo, entries=entries)


def gather_profiles(local: dict, n_stages: int) -> list:
    """All ranks end with the same profile list (stage order)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, {k: dict(v.entries) for k, v in local.items()})
        merged = {}
        for p in parts:
            merged.update(p)
        layers = {k: v.layers for k, v in local.items()}
        lay_parts = [None] * dist.get_world_size()
        dist.all_gather_object(lay_parts, layers)
        for p in lay_parts:
            layers.update(p)
        return [pipelink.StageProfile(stage_id=s, layers=layers[s], entries=merged[s])
                for s in range(n_stages)]
    return [local[s] for s in range(n_stages)]


def measure_links(engine, small: int = 4096, large: int = 16 << 20, reps: int = 5) -> list:
    """Measure every hop of `engine` as a reference LinkProfile (latency_s, bytes/s).

    Same-process hops time a device copy on the source's link stream; hops between
    ranks time an ncclSend on the source rank's link communicator (the matching
    ncclRecv is posted by the destination).  latency = time(small message);
    bandwidth = (large - small) / (time(large) - time(small)).  All ranks iterate
    the hops in the same order and the results are all-gathered, so every rank's
    virtual clock sees identical link profiles.
    """
    import torch.distributed as dist

    from . import _native as N

    g = engine.gpu
    pl = g.pl
    S = pl.n_stages
    lib = N.lib()
    measured = {}
    if S < 2:
        return []
    for link in range(S):
        src = S - 1 if link == S - 1 else link
        dst = 0 if link == S - 1 else link + 1
        src_local, dst_local = pl.local(src), pl.local(dst)
        if not (src_local or dst_local):
            continue
        dev = g.exe[src].device if src_local else g.exe[dst].device
        with torch.cuda.device(dev):
            sbuf = torch.empty(large, dtype=torch.uint8, device=dev) if src_local else None
            dbuf = (torch.empty(large, dtype=torch.uint8, device=g.exe[dst].device)
                    if dst_local else None)
            st = torch.cuda.Stream(dev)  # a private link stream (the runtime's are C++-owned)

            def once(nbytes):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                if src_local and dst_local:
                    N.check(lib.pl_memcpy_async(dbuf.data_ptr(), sbuf.data_ptr(), nbytes, st.cuda_stream),
                            "pl_memcpy_async")
                elif src_local:
                    N.check(lib.pl_p2p_send(g.comms[link], sbuf.data_ptr(), nbytes, 1, st.cuda_stream),
                            "pl_p2p_send")
                else:
                    N.check(lib.pl_p2p_recv(g.comms[link], dbuf.data_ptr(), nbytes, 0, st.cuda_stream),
                            "pl_p2p_recv")
                b.record(st)
                b.synchronize()
                return a.elapsed_time(b) / 1e3

            once(small)
            t_small = float(np.median([once(small) for _ in range(reps)]))
            t_large = float(np.median([once(large) for _ in range(reps)]))
        if src_local:
            bw = (large - small) / max(t_large - t_small, 1e-9)
            measured[link] = (round(t_small, 9), float(f"{bw:.4g}"))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, measured)
        for p in parts:
            measured.update(p)
    out = []
    for link, lp in enumerate(engine.link_profiles):
        lat, bw = measured[link]
        out.append(pipelink.LinkProfile(lp.src, lp.dst, lat, bw))
    return out
