"""CPU reproduction: the reference controller's n = 6 / n = 7 split at S = 8.

    python scripts/controller_bimodal.py

Runs the unmodified ``pipelink.PipelineEngine`` (virtual clock, no GPU) on the
8-stage Llama-3-8B-shape deployment of ``scripts/run_stages.py`` with the stage
and link profiles MEASURED by repeated runs of that script
(``profiles/r2/multigpu/s8_profiles_rep*.log``, full tables at full precision).
Prints, per run, the decision counts and the virtual span: the two measured
tables differ by ~1 % yet put the reference's greedy ``choose_n`` on different
n, and the n = 7 schedule is about twice as long in the reference's own clock.
"""

import json
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_05043_b200 import PRESETS, deploy  # noqa: E402  (locates pipelink)
import pipelink as PL  # noqa: E402


def run(log: Path):
    d = json.loads([l for l in log.read_text().splitlines() if l.startswith("{")][-1])
    spec = PRESETS["llama3-8b-shape"]
    S = len(d["stage_decode_profiles_ms"])
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    ctrl = PL.ControllerConfig(max_batched_tokens=32768, max_batch_size=64)
    cfg = deploy.engine_config(plan, spec, ctrl)
    profiles = [PL.StageProfile(stage_id=s, layers=p["layers"],
                                entries={(PL.Phase[ph], int(t)): v for ph, t, v in p["entries"]})
                for s, p in enumerate(d["stage_profiles"])]
    eng = PL.PipelineEngine(cfg, cluster, profiles)
    eng.link_profiles = [PL.LinkProfile(a, b, lat, bw) for a, b, lat, bw in d["link_profiles"]]
    res = eng.run(deploy.uniform_trace(64, 512, 256))
    counts = Counter(dec.n_microbatches for _, dec in res.decisions)
    return {"log": log.name, "device_run": {"decisions": d.get("decision_counts"), "virtual_span_s": d["virtual_span_s"]},
            "reference_cpu": {"decisions": dict(sorted(counts.items())), "virtual_span_s": round(res.end_ns / 1e9, 4)}}


if __name__ == "__main__":
    for name in sys.argv[1:] or ("s8_profiles_rep1.log", "s8_profiles_rep2.log", "s8_profiles_rep3.log"):
        print(json.dumps(run(ROOT / "profiles" / "r2" / "multigpu" / name)))
