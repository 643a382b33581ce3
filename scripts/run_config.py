"""Run BASELINE configs 3-5 on the B200 pipeline and print one JSON summary line.

  config 4  mixed contention: 64 decoders (512/256) at t=0, 8 x 2048-token prompts
            (output 16) arriving during decode; prefill chunking on vs off;
            NVLink or 100 Mbps / 15 ms throttled links.
  config 5  weak-link emulation: 8-stage Llama-3-8B shape, every hop throttled to
            100 Mbps + 15 ms one-way, 64 requests 512/32, dynamic (n_max=None) vs
            static (n_max=S) micro-batching: per-stage bubbles and tok/s.
  config 3  Qwen2-72B shape, 8 stages, 256 requests (512/256 assumed), dynamic n,
            max_batched_tokens 131072 (needs >= 4 GPUs: torchrun, 2 stages/GPU).

    python scripts/run_config.py --config 5 [--decode 32] [--stages 8]
    torchrun --nproc-per-node 4 scripts/run_config.py --config 3
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[3, 4, 5])
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--decode", type=int, default=0)
    ap.add_argument("--throttle", action="store_true")
    ap.add_argument("--variants", default="")
    ap.add_argument("--layers", type=int, default=0)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend="cuda:nccl,cpu:gloo")

    from paper_2507_05043_b200 import LLAMA3_8B, QWEN2_72B, deploy
    from paper_2507_05043_b200.engine import B200PipelineEngine
    from paper_2507_05043_b200.profiler import gather_profiles, profile_stage
    import pipelink as PL

    if a.config == 3:
        spec, S, B, dec = QWEN2_72B, a.stages or 8, a.batch or 256, a.decode or 256
        mbt, variants = 131072, [("dynamic", None, PL.DEFAULT_CHUNK_SIZE)]
        link = deploy.NVLINK
    elif a.config == 4:
        spec, S, B, dec = LLAMA3_8B, a.stages or 4, a.batch or 64, a.decode or 256
        mbt = 32768
        variants = [("chunked", None, PL.DEFAULT_CHUNK_SIZE), ("unchunked", None, None)]
        link = deploy.WEAK_LINK if a.throttle else deploy.NVLINK
    else:
        spec, S, B, dec = LLAMA3_8B, a.stages or 8, a.batch or 64, a.decode or 32
        mbt = 32768
        variants = [("dynamic", None, PL.DEFAULT_CHUNK_SIZE), ("static", "S", PL.DEFAULT_CHUNK_SIZE)]
        link = deploy.WEAK_LINK
        a.throttle = True
    if a.layers:
        spec = spec.with_(num_layers=a.layers)
    if a.variants:
        keep = a.variants.split(",")
        variants = [v for v in variants if v[0] in keep]

    cluster = deploy.b200_cluster(S, *link)
    plan = deploy.plan(cluster, spec, S)
    reqs = [PL.Request(i, 0.0, a.prompt, dec) for i in range(B)]
    if a.config == 4:
        # 8 long prompts arrive while the decoders are mid-stream
        reqs += [PL.Request(B + i, 0.25 + 0.05 * i, 2048, 16) for i in range(8)]
    trace = PL.Trace(requests=reqs)

    results = {}
    eng = None
    for name, n_max, chunk in variants:
        ctrl = PL.ControllerConfig(max_batched_tokens=mbt, max_batch_size=max(B, 64),
                                   n_max=(S if n_max == "S" else n_max))
        cfg = deploy.engine_config(plan, spec, ctrl, chunk_size=chunk)
        placeholder = [PL.synth_profile(hi - lo, 1e-6, 1e-4, stage_id=i)
                       for i, (_, (lo, hi)) in enumerate(plan.stages)]
        t0 = time.time()
        eng = B200PipelineEngine(cfg, cluster, placeholder, decoder=spec, throttle=a.throttle)
        eng.prepare(trace)
        prof = gather_profiles({s: profile_stage(x, ctx=a.prompt) for s, x in eng.gpu.exe.items()}, S)
        eng.set_stage_profiles(prof)
        # warm-up on a 4-request slice of the trace: NCCL connections, TMA descriptor
        # caches and first launches are paid outside the measured run
        warm = PL.Trace(requests=[PL.Request(r.id, 0.0, min(r.input_len, 256), 2)
                                  for r in trace.requests[:4]])
        eng.run(warm)
        setup = time.time() - t0
        w0 = time.perf_counter()
        res = eng.run(trace)
        wall = time.perf_counter() - w0
        run_s = res.b200.run_time_s
        if world > 1:
            t = torch.tensor([run_s, wall], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            run_s, wall = t.tolist()
        span = res.end_ns / 1e9
        bubbles = [round(PL.measure_bubble(res, s, 0.0, span), 5) for s in range(S)]
        rep = PL.summarize(res.requests, tuple(bubbles))
        out = {"virtual_tok_s": round(rep.throughput_tok_s, 2), "virtual_span_s": round(span, 4),
               "virtual_bubbles": bubbles, "device_run_s": round(run_s, 4), "wall_s": round(wall, 3),
               "device_tok_s": round(sum(r.tokens_emitted for r in res.requests) / run_s, 2),
               "decisions_n": sorted({d.n_microbatches for _, d in res.decisions}),
               "setup_s": round(setup, 1), "all_finished": res.all_finished}
        if rank == 0 and res.b200.token_times_s:
            gaps = []
            for rid, ts in res.b200.token_times_s.items():
                if rid < B:
                    gaps += [b - c for c, b in zip(ts, ts[1:])]
            gaps.sort()
            if gaps:
                out["decode_inter_token_p50_ms"] = round(1e3 * gaps[len(gaps) // 2], 3)
                out["decode_inter_token_p99_ms"] = round(1e3 * gaps[min(len(gaps) - 1, int(0.99 * len(gaps)))], 3)
            out["tpot_p50_ms"] = round(1e3 * (res.b200.tpot_p50_s() or 0), 3)
        # max decode wait on any link (virtual link log: first emit - enqueue)
        enq, emit = {}, {}
        for e in res.link_events:
            if e.phase_class is PL.PayloadClass.DECODE:
                key = (e.link, e.payload_id)
                if e.event == "enqueue":
                    enq[key] = e.time_ns
                elif e.event == "emit" and key not in emit:
                    emit[key] = e.time_ns
        waits = [emit[k] - enq[k] for k in emit if k in enq]
        out["max_decode_link_wait_ms"] = round(max(waits) / 1e6, 3) if waits else None
        results[name] = out
        eng.close()
        del eng
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"config": a.config, "model": spec.name, "stages": S, "gpus": world,
                          "batch": B, "prompt": a.prompt, "decode": dec, "throttle": a.throttle,
                          "link": {"latency_s": link[0], "bandwidth_Bps": link[1]},
                          "results": results}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
