"""B200PipelineEngine: the drop-in for ``pipelink.PipelineEngine`` with real compute and links.

    from pipelink import EngineConfig, ControllerConfig, ...      # unchanged reference API
    from paper_2507_05043_b200 import B200PipelineEngine, LLAMA3_8B

    engine = B200PipelineEngine(cfg, cluster, stage_profiles, decoder=LLAMA3_8B)
    result = engine.run(trace)          # pipelink.RunResult, schedule == PipelineEngine's
    result.b200.tokens[rid]             # greedy token ids generated on the GPUs
    result.b200.decode_tok_s            # measured on the device clock

Same constructor arguments and ``run(trace, horizon_s)`` contract as the
reference (engine.py:264-294, 509-600), plus the decoder shape the reference
cannot know (its ModelSpec has no heads/FFN/vocab).  Under ``torchrun`` each
rank constructs the engine identically and owns ``S / world_size`` contiguous
stages; hops between ranks are NCCL P2P.

By default (``native=True``) ``run`` hands the whole event loop to the C++
scheduler (csrc/sched.cu), whose hooks issue every per-micro-batch GPU action
in C++ (csrc/runtime.cu); ``native=False`` runs the Python twin
(driver.PipelineDriver + backend.GpuBackend).  Both give the identical
schedule and tokens.  Extra keywords: ``throttle=True`` replays the virtual
link timing on the GPU clock; ``prompts={rid: ids}`` overrides the synthetic
prompts; ``devices=[...]`` spreads stages over local GPUs without torchrun;
``fuse_transport`` (opt-in, native runtime) stores decode payloads between
stages of this process from the producer's last residual epilogue straight into
the next stage's buffer over NVLink peer memory instead of a link copy (measured
slower across GPUs: the producer then waits on the consumer's slot).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._pipelink import pipelink
from .backend import GpuBackend, Placement
from .driver import PipelineDriver
from .spec import DecoderSpec

nearest_rank = pipelink.metrics.nearest_rank


@dataclass
class B200Stats:
    """Device-clock measurements of one run (rank-local; tokens on the head rank)."""

    run_time_s: float
    tokens: dict | None = None          # rid -> np.ndarray of generated ids (head rank)
    token_times_s: dict | None = None   # rid -> device time of each emitted token
    decode_start_s: float | None = None
    total_tokens: int = 0
    decode_tokens: int = 0
    real: object = None                 # pipelink RunResult on the device clock
    extra: dict = field(default_factory=dict)

    @property
    def throughput_tok_s(self) -> float:
        return self.total_tokens / self.run_time_s if self.run_time_s > 0 else 0.0

    @property
    def decode_time_s(self) -> float | None:
        if self.decode_start_s is None:
            return None
        return self.run_time_s - self.decode_start_s

    @property
    def decode_tok_s(self) -> float | None:
        t = self.decode_time_s
        return self.decode_tokens / t if t else None

    def tpot_p50_s(self) -> float | None:
        if not self.token_times_s:
            return None
        tp = sorted((ts[-1] - ts[0]) / (len(ts) - 1) for ts in self.token_times_s.values() if len(ts) >= 2)
        return nearest_rank(tp, 50) if tp else None

    def ttft_p50_s(self) -> float | None:
        if not self.token_times_s:
            return None
        return nearest_rank(sorted(ts[0] for ts in self.token_times_s.values()), 50)


def schedule_key(res) -> dict:
    """Everything the reference scheduler decides in a RunResult (engine.py:108-127): event
    log, link log (chunk boundaries and times), controller decisions, busy intervals,
    token emissions and request lifecycles.  Two runs made the same schedule iff their
    keys are equal."""
    return {
        "events": [(e.time_ns, int(e.kind), e.subject, e.stage) for e in res.events],
        "links": [(e.time_ns, e.link, e.payload_id, e.chunk_index, e.size_bytes, e.phase_class.value,
                   e.event) for e in res.link_events],
        "decisions": [(i, d.n_microbatches, d.token_budget_per_microbatch, d.predicted_bubble_fraction)
                      for i, d in res.decisions],
        "busy": res.stage_busy_ns,
        "emissions": res.token_emissions,
        "first": sorted(res.first_compute_ns.items()),
        "end": res.end_ns,
        "done": res.all_finished,
        "reqs": [(r.id, r.state.value, r.tokens_emitted, r.first_token_time, r.finish_time,
                  r.arrival_time) for r in res.requests],
    }


def create_link_comms(placement: Placement) -> dict:
    """One 2-rank NCCL communicator per directed hop whose stages sit on different ranks.
    Unique ids travel over the default torch.distributed group (rendezvous only)."""
    import torch.distributed as dist

    S = placement.n_stages
    comms = {}
    if S < 2:
        return comms
    me = placement.rank
    for link in range(S):
        src = S - 1 if link == S - 1 else link
        dst = 0 if link == S - 1 else link + 1
        ra, rb = placement.stage_rank[src], placement.stage_rank[dst]
        if ra == rb:
            continue
        obj = [None]
        if me == ra:
            buf = (C.c_uint8 * 128)()
            N.call("pl_nccl_unique_id", buf, 128)
            obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=ra)
        if me in (ra, rb):
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            h = C.c_void_p()
            N.call("pl_comm_init_rank", uid, 2, 0 if me == ra else 1, C.byref(h))
            comms[link] = h
    return comms


class B200PipelineEngine(PipelineDriver):
    """``native=True`` (default): the event loop and every per-micro-batch GPU action
    run in C++ (NativeScheduler + pl_pipeline); ``native=False``: the Python
    PipelineDriver + GpuBackend twin.  Both produce the identical schedule."""

    def __init__(self, cfg, cluster, stage_profiles, *, decoder: DecoderSpec, seed: int = 0,
                 devices: list | None = None, prompts: dict | None = None, throttle: bool = False,
                 native: bool = True, fuse_transport: bool = False):
        if cfg.model.hidden_dim != decoder.d or cfg.model.dtype_bytes != 2:
            raise pipelink.ConfigError("cfg.model must describe the decoder's bf16 residual stream "
                                       "(use DecoderSpec.model_spec())")
        if cfg.partition.num_layers != decoder.num_layers:
            raise pipelink.ConfigError("partition layer count != decoder layers")
        S = len(cfg.partition.stages)
        world, rank = 1, 0
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            world, rank = torch.distributed.get_world_size(), torch.distributed.get_rank()
        self.placement = Placement(S, world, rank, devices)
        local = sorted({d.index for d in self.placement.stage_device if d is not None and d.index is not None})
        if len(local) > 1:  # same-process hops between GPUs: direct NVLink peer copies
            arr = (C.c_int32 * len(local))(*local)
            N.call("pl_enable_peer_access", len(local), arr)
        comms = create_link_comms(self.placement) if world > 1 else {}
        self.gpu = GpuBackend(decoder, cfg, self.placement, seed=seed, prompts=prompts, comms=comms,
                              throttle=throttle)
        self.gpu.fuse_transport = fuse_transport
        super().__init__(cfg, cluster, stage_profiles, backend=self.gpu)
        self._comms = comms
        self.native = native
        self._sched = None

    def set_stage_profiles(self, stage_profiles) -> None:
        super().set_stage_profiles(stage_profiles)
        self._sched = None

    def set_link_profiles(self, link_profiles) -> None:
        super().set_link_profiles(link_profiles)
        self._sched = None

    def _native_run(self, trace, horizon_s):
        from .native import NativeScheduler

        if self._sched is None:
            self._sched = NativeScheduler(self.cfg, self.stage_profiles, self.link_profiles,
                                          self.bytes_per_token)
        g = self.gpu
        g.driver = self
        handle = g.native_start(trace, record_links=g.record_links)
        result = self._sched.run(trace, horizon_s, pipeline=handle)
        g.native_finish(result)
        return result

    def run(self, trace, horizon_s: float | None = None):
        if self.native:
            result = self._native_run(trace, horizon_s)
        else:
            result = super().run(trace, horizon_s)
        g = self.gpu
        stats = B200Stats(run_time_s=g.run_time_s, tokens=g.tokens, decode_start_s=g.decode_start_s)
        if g.tokens is not None:
            times: dict = {}
            for t, (ev, rids) in zip(g.fb_times_s, g.fb_events):
                for rid in rids:
                    times.setdefault(rid, []).append(t)
            stats.token_times_s = times
            stats.total_tokens = sum(len(v) for v in g.tokens.values())
            stats.decode_tokens = sum(max(0, len(v) - 1) for v in g.tokens.values())
        stats.real = self._real_result(result)
        result.b200 = stats
        return result

    def _real_result(self, virtual):
        """The run re-expressed on the device clock as a reference RunResult, so the
        unchanged summarize() / measure_bubble() (metrics.py:78-117, engine.py:130-144)
        report measured TTFT/TPOT/throughput/bubbles.  Stage intervals cover this
        rank's stages; token times exist on the head rank.  The device replay does not
        pace arrivals, so a request "arrives" on the device clock when its first
        micro-batch starts on stage 0: device TTFT is dispatch to first token."""
        g = self.gpu
        S = len(self.stage_profiles)
        busy = [[(a, b) for _, a, b in g.busy_real_ns.get(s, [])] for s in range(S)]
        first_compute = {}
        for mb_id, a, _ in g.busy_real_ns.get(0, []):
            for rid in g.mb_requests.get(mb_id, ()):
                first_compute[rid] = min(a, first_compute.get(rid, a))
        emissions = []
        reqs = []
        times = {}
        if g.tokens is not None:
            for t, (_, rids) in zip(g.fb_times_s, g.fb_events):
                for rid in rids:
                    emissions.append((round(t * 1e9), rid))
                    times.setdefault(rid, []).append(t)
        for r in virtual.requests:
            c = r.fresh_copy()
            c.arrival_time = first_compute[r.id] / 1e9 if r.id in first_compute else r.arrival_time
            c.state, c.tokens_emitted = r.state, r.tokens_emitted
            ts = times.get(r.id)
            if ts:
                c.first_token_time, c.finish_time = ts[0], ts[-1]
            reqs.append(c)
        end_ns = round(g.run_time_s * 1e9)
        return pipelink.engine.RunResult(
            requests=reqs, events=[], link_events=[], decisions=virtual.decisions, stage_busy_ns=busy,
            token_emissions=sorted(emissions), first_compute_ns=first_compute, end_ns=end_ns,
            all_finished=virtual.all_finished)

    def prepare(self, trace) -> None:
        """Allocate weights, KV cache and buffers for `trace` ahead of the first run."""
        self.gpu.prepare(trace)

    def close(self) -> None:
        if self._sched is not None:
            self._sched.close()
            self._sched = None
        self.gpu.close()
        for h in self._comms.values():
            N.lib().pl_comm_destroy(h)
        self._comms = {}
