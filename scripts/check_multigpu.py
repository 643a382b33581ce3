"""Multi-GPU parity check (run under torchrun, one rank per GPU).

    torchrun --nproc-per-node 2 scripts/check_multigpu.py [--stages 2] [--model tiny]

Every rank builds the same B200PipelineEngine; stages are split over the ranks
and hops between ranks are NCCL P2P.  Rank 0 (the head) checks that the greedy
ids equal the CPU oracle's and that the schedule equals pipelink's.  Every rank
measures its links (profiler.measure_links: NCCL send timing, fed to the
controller), records the realized per-chunk NCCL log of the links it sends on
(CUDA events around each ncclSend) and checks it against the virtual LinkQueue
log (tests/link_checks.py, after pkg/tests/test_transport.py:136-211).  One JSON
summary line on rank 0.  Exit code 0 = parity holds.
"""

import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--requests", type=int, default=8)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--decode", type=int, default=32)
    ap.add_argument("--chunk", type=int, default=262144)
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    from paper_2507_05043_b200.backend import local_device_index

    torch.cuda.set_device(local_device_index())
    dist.init_process_group(backend="cuda:nccl,cpu:gloo")

    from paper_2507_05043_b200 import LLAMA3_8B, TINY, deploy
    from paper_2507_05043_b200.engine import B200PipelineEngine
    from paper_2507_05043_b200.spec import prompt_tokens
    import pipelink as PL

    spec = {"tiny": TINY, "l3-2": LLAMA3_8B.with_(num_layers=2 * (a.stages or world))}[a.model]
    spec = spec.with_(peaked=True)
    S = a.stages or world
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    cfg = deploy.engine_config(plan, spec, PL.ControllerConfig(max_batched_tokens=1024,
                                                                max_batch_size=a.requests),
                               chunk_size=a.chunk or None)
    trace = deploy.uniform_trace(a.requests, a.prompt, a.decode)
    profiles = [PL.synth_profile(hi - lo, 1e-6, 2e-5, stage_id=i) for i, (_, (lo, hi)) in enumerate(plan.stages)]
    eng = B200PipelineEngine(cfg, cluster, profiles, decoder=spec)
    eng.run(PL.Trace(requests=[PL.Request(0, 0.0, 16, 2)]))  # NCCL connections, first launches
    from paper_2507_05043_b200.profiler import measure_links
    from link_checks import check_realized_link

    links = measure_links(eng)
    eng.set_link_profiles(links)
    eng.gpu.record_links = True
    res = eng.run(trace)
    ok = True
    refe = PL.PipelineEngine(cfg, cluster, profiles)
    refe.link_profiles = list(links)
    ref = refe.run(trace)
    if [(e.time_ns, e.kind, e.subject, e.stage) for e in res.events] != \
       [(e.time_ns, e.kind, e.subject, e.stage) for e in ref.events]:
        print(f"rank {rank}: schedule differs from pipelink", flush=True)
        ok = False
    link_report, link_err = {}, None
    try:
        for lp in links:
            if any(e.link == lp.name for e in eng.gpu.realized_links):
                link_report[lp.name] = check_realized_link(eng.gpu.realized_links, res.link_events, lp.name)
    except AssertionError as e:
        link_err = f"rank {rank}: {e}"
        ok = False
    parts = [None] * world
    dist.all_gather_object(parts, {"links": link_report, "err": link_err})
    if rank == 0:
        from oracle import decoder as OD

        model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=a.prompt + a.decode + 8)
        prompts = [torch.from_numpy(prompt_tokens(0, r.id, r.input_len, spec.vocab)) for r in trace.requests]
        want, _ = model.greedy(prompts, a.decode)
        bad = [r.id for i, r in enumerate(trace.requests)
               if not np.array_equal(res.b200.tokens[r.id], want[i].numpy())]
        print(f"world {world}, {S} stages: {len(trace.requests) - len(bad)}/{len(trace.requests)} requests "
              f"identical to the CPU oracle; device {res.b200.run_time_s * 1e3:.1f} ms", flush=True)
        import json

        realized = {}
        for p in parts:
            realized.update(p["links"])
        print(json.dumps({"world": world, "stages": S, "model": a.model, "tokens_identical": not bad,
                          "schedule_equal": ok, "nccl_max_nchannels": os.environ.get("NCCL_MAX_NCHANNELS"),
                          "measured_links": [{"name": lp.name, "latency_us": round(lp.latency_s * 1e6, 2),
                                              "bandwidth_GBps": round(lp.bandwidth_bps / 1e9, 1)} for lp in links],
                          "realized_nccl_links": realized,
                          "link_errors": [p["err"] for p in parts if p["err"]],
                          "device_run_ms": round(res.b200.run_time_s * 1e3, 2)}), flush=True)
        ok = ok and not bad
    t = torch.tensor([0 if ok else 1])
    dist.all_reduce(t)
    eng.close()
    dist.destroy_process_group()
    sys.exit(int(t.item() != 0))


if __name__ == "__main__":
    main()
