"""S pipeline stages on G local GPUs in ONE process (peer copies over NVLink).

    python scripts/run_stages.py --stages 8 --gpus 4        (gpurun --gpus 4)
    python scripts/run_stages.py --stages 8 --gpus 1

The north-star shape (Llama-3-8B, 8 stages, B=64, 512/256) on fewer GPUs than stages:
stages are placed contiguously (two per GPU on 4 GPUs), every hop between GPUs is a
cudaMemcpyAsync peer copy on the source stage's link stream, same-GPU hops are device
copies.  Reports, on the device clock:
* decode-window tok/s and the SURVEY §8(d) roofline computed PER GPU (stages that
  share a GPU share its HBM: their bytes add), plus the 8-independent-GPU roofline for
  reference; frac = achieved / per-GPU roofline;
* measured link profiles (profiler.measure_links) fed to the controller;
* schedule equality with pipelink.PipelineEngine on the same profiles;
* the realized per-chunk link log checked against the virtual one (tests/link_checks.py).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def per_gpu_roofline(spec, eng, hbm_gbs, tflops, stage_gpu):
    plan = eng.cfg.partition
    S = len(plan.stages)
    layer_b = spec.layer_bytes()
    head_b = spec.vocab * spec.d * 2 + spec.d * 2
    kv_tl = spec.kv_bytes_per_token_layer()
    per_stage = [0.0] * S
    tokens = 0
    for phase, R, ctx_sum in eng.gpu.mb_log:
        if phase != "decode":
            continue
        tokens += R
        for s, (_, (lo, hi)) in enumerate(plan.stages):
            L = hi - lo
            wb = L * layer_b + (head_b if s == S - 1 else 0)
            flops = 2 * R * (L * spec.layer_params() + (spec.vocab * spec.d if s == S - 1 else 0))
            per_stage[s] += max((wb + ctx_sum * L * kv_tl) / (hbm_gbs * 1e9), flops / (tflops * 1e12))
    gpus = sorted(set(stage_gpu))
    per_gpu = {g: sum(t for s, t in enumerate(per_stage) if stage_gpu[s] == g) for g in gpus}
    t_gpu, t_stage = max(per_gpu.values()), max(per_stage)
    return {"decode_tokens": tokens, "per_gpu_roofline_tok_s": round(tokens / t_gpu, 1),
            "independent_gpu_roofline_tok_s": round(tokens / t_stage, 1),
            "binding_gpu": max(per_gpu, key=per_gpu.get), "binding_stage": per_stage.index(t_stage),
            "stage_roofline_ms": [round(t * 1e3, 2) for t in per_stage]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="llama3-8b-shape")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--decode", type=int, default=256)
    ap.add_argument("--max-batched", type=int, default=32768, help="controller max_batched_tokens")
    ap.add_argument("--no-links", action="store_true", help="skip the realized link log")
    ap.add_argument("--fuse", action="store_true", help="store decode payloads from the producer's epilogue")
    a = ap.parse_args()

    import torch

    from paper_2507_05043_b200 import PRESETS, deploy  # locates the reference pipelink first
    import bench as B
    import pipelink as PL
    from link_checks import check_realized_link
    from paper_2507_05043_b200.engine import B200PipelineEngine, schedule_key
    from paper_2507_05043_b200.profiler import measure_links, profile_stage

    spec = PRESETS[a.model]
    if a.layers:
        spec = spec.with_(num_layers=a.layers)
    S, G = a.stages, a.gpus
    devices = [torch.device("cuda", g) for g in range(G)]
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    ctrl = PL.ControllerConfig(max_batched_tokens=a.max_batched, max_batch_size=a.batch)
    cfg = deploy.engine_config(plan, spec, ctrl)
    trace = deploy.uniform_trace(a.batch, a.prompt, a.decode)
    placeholder = [PL.synth_profile(hi - lo, 1e-6, 1e-4, stage_id=i) for i, (_, (lo, hi)) in enumerate(plan.stages)]
    t0 = time.time()
    eng = B200PipelineEngine(cfg, cluster, placeholder, decoder=spec, devices=devices,
                             fuse_transport=a.fuse)
    eng.prepare(trace)
    eng.set_stage_profiles([profile_stage(eng.gpu.exe[s], ctx=a.prompt) for s in range(S)])
    warm = PL.Trace(requests=[PL.Request(r.id, 0.0, min(r.input_len, 256), 2) for r in trace.requests[:4]])
    eng.run(warm)  # streams, NCCL-free peer paths, descriptor caches
    links = measure_links(eng)
    eng.set_link_profiles(links)
    setup = time.time() - t0
    eng.gpu.record_links = not a.no_links
    hbm, tfl, _ = B.peaks()
    with B.ClockSampler(0) as clk:
        w0 = time.perf_counter()
        res = eng.run(trace)
        wall = time.perf_counter() - w0
    st = res.b200
    dec_t = st.decode_time_s
    window = (a.batch * (a.decode - 1)) / dec_t if dec_t else None
    stage_gpu = [eng.placement.stage_device[s].index for s in range(S)]
    roof = per_gpu_roofline(spec, eng, hbm, tfl, stage_gpu)
    ref = PL.PipelineEngine(cfg, cluster, eng.stage_profiles)
    ref.link_profiles = list(eng.link_profiles)
    vres = ref.run(trace)
    ka, kb = schedule_key(vres), schedule_key(res)
    link_report = {}
    if not a.no_links:
        for lp in eng.link_profiles:
            link_report[lp.name] = check_realized_link(eng.gpu.realized_links, res.link_events, lp.name)
    span = res.end_ns / 1e9
    bubbles = [round(PL.measure_bubble(st.real, s, 0.0, st.real.end_ns / 1e9), 4) for s in range(S)]
    out = {"workload": f"{spec.name} {S}-stage pipeline on {G} GPU(s), one process, {a.batch} requests "
                       f"{a.prompt}/{a.decode}",
           "stage_gpu": stage_gpu, "fused_transport": a.fuse,
           "device_tok_s": round(st.throughput_tok_s, 1),
           "decode_window_tok_s": round(window, 1) if window else None,
           "tpot_p50_ms": round(1e3 * (st.tpot_p50_s() or 0), 3), "ttft_p50_ms": round(1e3 * (st.ttft_p50_s() or 0), 2),
           "roofline": roof,
           "frac_of_per_gpu_roofline": round(window / roof["per_gpu_roofline_tok_s"], 4) if window else None,
           "frac_of_independent_gpu_roofline": round(window / roof["independent_gpu_roofline_tok_s"], 4)
           if window else None,
           "measured_links": [{"name": lp.name, "latency_us": round(lp.latency_s * 1e6, 2),
                               "bandwidth_GBps": round(lp.bandwidth_bps / 1e9, 1)} for lp in links],
           "schedule_equal_pipelink": ka == kb, "virtual_span_s": round(span, 4),
           "device_stage_bubbles": bubbles,
           "decisions_n": sorted({d.n_microbatches for _, d in res.decisions}),
           "decision_counts": {str(n): sum(1 for _, d in res.decisions if d.n_microbatches == n)
                               for n in sorted({d.n_microbatches for _, d in res.decisions})},
           # the measured decode tables the controller decided on (ms at T tokens)
           "stage_decode_profiles_ms": [{str(t): round(v * 1e3, 4) for (ph, t), v in sorted(p.entries.items(),
                                                                                          key=lambda kv: kv[0][1])
                                         if ph is PL.Phase.DECODE} for p in eng.stage_profiles],
           # full tables at full precision (scripts/controller_bimodal.py replays them on the CPU)
           "stage_profiles": [{"layers": p.layers, "entries": [[ph.name, t, v] for (ph, t), v in p.entries.items()]}
                              for p in eng.stage_profiles],
           "link_profiles": [[lp.src, lp.dst, lp.latency_s, lp.bandwidth_bps] for lp in eng.link_profiles],
           "realized_links": link_report or None, "clocks": clk.summary, "wall_s": round(wall, 2),
           "setup_s": round(setup, 1)}
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
