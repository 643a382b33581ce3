"""``pipelink simulate`` with ``--backend b200``: the reference's run config, real compute.

    python -m paper_2507_05043_b200.cli simulate --config run.json --out outdir \\
        [--backend b200|virtual] [--decoder llama3-8b-shape] [--measure-profiles] [--throttle]

The reference CLI's simulate (pipelink/cli.py:224-255) assembles cluster, plan,
trace, profiles and engine config from a JSON run config, runs ``PipelineEngine``
and writes report.json / events.csv / transport.csv / decisions.csv.  This entry
point reuses every one of those steps from the reference module unchanged and
swaps only the engine: ``B200PipelineEngine`` executes the same schedule on the
GPUs of this box (one stage per GPU when there are enough, else stages spread over
the visible GPUs in one process).  The virtual outputs are the reference's (the
schedule is identical); ``b200.json`` adds the device-clock report --
``summarize``/``measure_bubble`` of the measured run -- and the generated tokens.

The decoder shape comes from ``--decoder`` or the run config's extra key
``"decoder"`` (the reference's ModelSpec has no heads / FFN / vocabulary);
``--measure-profiles`` replaces the config's stage profiles with ones measured on
the B200s (profiler.profile_stage) before the run.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from ._pipelink import pipelink


def _ref_cli():
    import importlib

    return importlib.import_module("pipelink.cli")


def run_b200(cfg, args):
    import torch

    from . import PRESETS
    from .engine import B200PipelineEngine
    from .profiler import profile_stage

    C = _ref_cli()
    cluster = C.load_cluster(cfg.cluster_path)
    plan = C.plan_deployment(cluster, cfg.model, cfg.gpu_type, cfg.gpu_count)
    trace = C._build_trace(cfg, args.seed)
    if not trace.requests:
        raise pipelink.ConfigError("trace is empty; nothing to simulate")
    profiles = C._build_profiles(cfg, plan, cluster)
    engine_cfg = C._build_engine_config(cfg, plan, args.seed)
    raw = json.loads(Path(args.config).read_text())
    name = args.decoder or raw.get("decoder")
    if name not in PRESETS:
        raise pipelink.ConfigError(f"--decoder (or the config's 'decoder') must be one of {sorted(PRESETS)}")
    spec = PRESETS[name]
    S = len(plan.stages)
    n = max(1, torch.cuda.device_count())
    devices = [torch.device("cuda", g) for g in range(min(n, S))]
    eng = B200PipelineEngine(engine_cfg, cluster, profiles, decoder=spec, devices=devices, throttle=args.throttle)
    if args.measure_profiles:
        eng.prepare(trace)
        eng.set_stage_profiles([profile_stage(eng.gpu.exe[s]) for s in range(S)])
    result = eng.run(trace)
    if not result.all_finished:
        raise pipelink.PipelinkError("run ended with unfinished requests")
    report = C._report_from_result(result)
    real = result.b200.real
    real_report = C._report_from_result(real)
    eng.close()
    return result, report, real_report


def cmd_simulate(args) -> int:
    C = _ref_cli()
    cfg = C.load_run_config(args.config)
    out = Path(args.out)
    if args.backend == "virtual":
        result, report, _ = C.run_simulation(cfg, args.seed)
        C._write_outputs(out, result, report)
        print(report.format_table())
        return 0
    result, report, real_report = run_b200(cfg, args)
    C._write_outputs(out, result, report)  # the schedule: identical to the reference engine's
    st = result.b200
    b200 = {"device_run_s": st.run_time_s, "device_tok_s": st.throughput_tok_s,
            "decode_tok_s": st.decode_tok_s, "tpot_p50_s": st.tpot_p50_s(), "ttft_p50_s": st.ttft_p50_s(),
            "device_report": json.loads(json.dumps(real_report.__dict__, default=str)),
            "tokens": {str(k): v.tolist() for k, v in (st.tokens or {}).items()}}
    (out / "b200.json").write_text(json.dumps(b200, indent=1) + "\n")
    print(report.format_table())
    print(f"device clock: {st.throughput_tok_s:.1f} tok/s over {st.run_time_s:.4f} s; outputs in {out}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="b200link")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sim = sub.add_parser("simulate", help="run a pipelink run config on the B200 backend")
    sim.add_argument("--config", required=True)
    sim.add_argument("--out", default="out")
    sim.add_argument("--seed", type=int, default=None)
    sim.add_argument("--backend", choices=["b200", "virtual"], default="b200")
    sim.add_argument("--decoder", default=None)
    sim.add_argument("--measure-profiles", action="store_true")
    sim.add_argument("--throttle", action="store_true", help="replay the virtual link timing on the GPU clock")
    args = ap.parse_args(argv)
    return cmd_simulate(args)


if __name__ == "__main__":
    sys.exit(main())
