"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

Each rank runs the deterministic driver on its own and issues only the work of
its stages (paper_2507_05043_b200.backend.Placement).  Correctness of the NCCL
data path rests on three host-side facts checked here with real processes:

1. every rank computes the identical schedule (no control messages exist);
2. for every directed hop, the sequence of (payload, chunk, byte offset, size)
   the source rank sends equals the sequence the destination rank receives,
   and the chunks tile each payload exactly -- so ncclSend/ncclRecv pairs match;
3. each rank's per-communicator issue order is a projection of one global
   order, which rules out cross-rank send/recv deadlock.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_05043_b200 import TINY, LLAMA3_8B, deploy
from paper_2507_05043_b200.backend import Placement
from paper_2507_05043_b200.driver import Backend, PipelineDriver

import pipelink


class RecordingBackend(Backend):
    """The GPU backend's routing decisions without a GPU: who computes, who sends what."""

    def __init__(self, placement: Placement):
        self.pl = placement
        self.ops = []          # (global seq, kind, link/stage, payload, chunk, offset, size)
        self.seq = 0

    def compute(self, stage, mb, now_ns):
        if self.pl.local(stage):
            self.ops.append((self.seq, "compute", stage, mb.id, -1, -1, mb.batched_tokens))
        self.seq += 1

    def emit(self, link, payload, chunk, offset, now_ns):
        S = self.pl.n_stages
        src = S - 1 if link == S - 1 else link
        dst = 0 if link == S - 1 else link + 1
        rec = (payload.id, chunk.index, offset, chunk.size_bytes, chunk.is_last, payload.size_bytes)
        if self.pl.local(src):
            self.ops.append((self.seq, "send", link, *rec[:4]))
        if self.pl.local(dst):
            self.ops.append((self.seq, "recv", link, *rec[:4]))
        self.seq += 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, S, spec_name, q):
    try:
        _work(rank, world, port, S, spec_name, q)
    except Exception as e:  # surface worker failures instead of a queue timeout
        q.put(repr(e))
        raise


def _work(rank, world, port, S, spec_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = {"tiny": TINY, "l3": LLAMA3_8B}[spec_name]
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    cfg = deploy.engine_config(plan, spec, pipelink.ControllerConfig(max_batched_tokens=4096,
                                                                       max_batch_size=16))
    profiles = [pipelink.synth_profile(hi - lo, 2e-6, 5e-5, stage_id=i)
                for i, (_, (lo, hi)) in enumerate(plan.stages)]
    trace = pipelink.Trace(requests=[pipelink.Request(i, 0.001 * (i // 5), 64 + 37 * i, 3 + i % 4)
                                     for i in range(24)])
    be = RecordingBackend(Placement(S, world, rank))
    res = PipelineDriver(cfg, cluster, profiles, backend=be).run(trace)
    digest = [(e.time_ns, int(e.kind), e.subject, e.stage) for e in res.events]
    out = [None] * world
    dist.all_gather_object(out, {"ops": be.ops, "digest": digest, "done": res.all_finished})
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def run_ranks(world, S, spec_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, spec_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    assert not isinstance(out, str), out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,S,spec", [(2, 2, "tiny"), (2, 4, "l3"), (4, 4, "l3"), (4, 8, "l3")])
def test_ranks_agree_and_p2p_pairs_match(world, S, spec):
    out = run_ranks(world, S, spec)
    # 1. identical schedules on every rank
    assert all(o["digest"] == out[0]["digest"] for o in out)
    assert all(o["done"] for o in out)
    pl = [Placement(S, world, r) for r in range(world)]
    for link in range(S):
        src = S - 1 if link == S - 1 else link
        dst = 0 if link == S - 1 else link + 1
        ra, rb = pl[0].stage_rank[src], pl[0].stage_rank[dst]
        sends = [op[3:] for op in out[ra]["ops"] if op[1] == "send" and op[2] == link]
        recvs = [op[3:] for op in out[rb]["ops"] if op[1] == "recv" and op[2] == link]
        # 2. matched pairs, in the same order, tiling each payload
        assert sends == recvs, f"link {link}: send/recv sequences differ"
        by_payload = {}
        for pid, idx, off, size in sends:
            by_payload.setdefault(pid, []).append((idx, off, size))
        for pid, chunks in by_payload.items():
            pos = 0
            for i, (idx, off, size) in enumerate(chunks):
                assert idx == i and off == pos
                pos += size
    # 3. each rank's issue order is increasing in the shared global sequence
    for o in out:
        seqs = [op[0] for op in o["ops"]]
        assert seqs == sorted(seqs)
    # every stage computed by exactly one rank
    computes = {}
    for r, o in enumerate(out):
        for op in o["ops"]:
            if op[1] == "compute":
                computes.setdefault((op[2], op[3]), []).append(r)
    assert all(len(v) == 1 for v in computes.values())
