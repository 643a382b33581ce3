"""Freeze the config-1 schedule golden under MEASURED profiles ("freeze the
real golden from measured profiles").

    python scripts/freeze_config1_golden.py measure [out.json]   # on a B200: stage + link profiles
    python scripts/freeze_config1_golden.py digest    # here: the reference engine's digests

`measure` builds BASELINE config 1 (tiny Llama, S = 2, 8 requests 128/32,
max_batched_tokens 1024) on one GPU, times both stages (profiler.profile_stage)
and the hop (profiler.measure_links), and writes tests/golden/config1_profiles.json.
`digest` runs the unmodified pipelink.PipelineEngine on those profiles and writes
the SHA-256 of every field of its RunResult (engine.schedule_key) to
tests/golden/config1_schedule.json; tests/test_config1_golden.py holds the
reference and the native scheduler to it.
"""

import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"

import paper_2507_05043_b200  # noqa: E402,F401  (puts the reference pipelink on the path)


def config1():
    import pipelink

    from paper_2507_05043_b200 import TINY, deploy

    cluster = deploy.b200_cluster(2)
    plan = deploy.plan(cluster, TINY, 2)
    ctrl = pipelink.ControllerConfig(max_batched_tokens=1024, max_batch_size=8)
    cfg = deploy.engine_config(plan, TINY, ctrl)
    return cfg, cluster, plan, deploy.uniform_trace(8, 128, 32)


def load_profiles():
    import pipelink

    d = json.loads((GOLD / "config1_profiles.json").read_text())
    phase = {p.value: p for p in pipelink.Phase}
    stages = [pipelink.StageProfile(stage_id=s["stage_id"], layers=s["layers"],
                                    entries={(phase[e[0]], e[1]): e[2] for e in s["entries"]})
              for s in d["stages"]]
    links = [pipelink.LinkProfile(l["src"], l["dst"], l["latency_s"], l["bandwidth_bps"]) for l in d["links"]]
    return stages, links


def cluster_with(cluster, links):
    import pipelink

    table = dict(cluster.links)
    for lp in links:
        table[(lp.src, lp.dst)] = lp
    return pipelink.ClusterSpec(nodes=cluster.nodes, links=table)


def digests(res) -> dict:
    from paper_2507_05043_b200.engine import schedule_key

    key = schedule_key(res)
    return {k: hashlib.sha256(json.dumps(v, default=str).encode()).hexdigest() for k, v in key.items()}


def measure():
    import torch

    from paper_2507_05043_b200 import TINY
    from paper_2507_05043_b200.engine import B200PipelineEngine
    from paper_2507_05043_b200.profiler import measure_links, profile_stage
    import pipelink

    cfg, cluster, plan, trace = config1()
    placeholder = [pipelink.synth_profile(hi - lo, 1e-6, 2e-5, stage_id=i)
                   for i, (_, (lo, hi)) in enumerate(plan.stages)]
    eng = B200PipelineEngine(cfg, cluster, placeholder, decoder=TINY, devices=[torch.device("cuda", 0)])
    eng.prepare(trace)
    stages = [profile_stage(eng.gpu.exe[s], ctx=128) for s in range(2)]
    links = measure_links(eng)
    eng.close()
    out = {"config": "BASELINE config 1: tiny Llama S=2, 8 requests 128/32, max_batched_tokens 1024",
           "measured_on": torch.cuda.get_device_name(0),
           "stages": [{"stage_id": p.stage_id, "layers": p.layers,
                       "entries": sorted([ph.value, t, sec] for (ph, t), sec in p.entries.items())}
                      for p in stages],
           "links": [{"src": lp.src, "dst": lp.dst, "latency_s": lp.latency_s, "bandwidth_bps": lp.bandwidth_bps}
                     for lp in links]}
    dst = Path(sys.argv[2]) if len(sys.argv) > 2 else GOLD / "config1_profiles.json"
    dst.parent.mkdir(parents=True, exist_ok=True)
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out)[:400])


def digest():
    import pipelink

    cfg, cluster, plan, trace = config1()
    stages, links = load_profiles()
    res = pipelink.PipelineEngine(cfg, cluster_with(cluster, links), stages).run(trace)
    out = {"profiles": "tests/golden/config1_profiles.json", "n_decisions": len(res.decisions),
           "n_events": len(res.events), "n_link_events": len(res.link_events),
           "tokens": len(res.token_emissions), "end_ns": res.end_ns, "sha256": digests(res)}
    (GOLD / "config1_schedule.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    {"measure": measure, "digest": digest}[sys.argv[1]]()
