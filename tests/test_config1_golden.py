"""BASELINE config 1's schedule frozen under MEASURED B200 profiles.

tests/golden/config1_profiles.json holds the stage and link profiles measured on a
B200 (scripts/freeze_config1_golden.py measure); config1_schedule.json the SHA-256 of
every RunResult field the unmodified pipelink.PipelineEngine produced with them
(... digest).  Both the reference engine (re-run here) and the native C++ scheduler
must reproduce every digest.
"""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "scripts"))

import freeze_config1_golden as F  # noqa: E402

GOLD = json.loads((ROOT / "tests" / "golden" / "config1_schedule.json").read_text())


def run_with(engine_cls_or_fn):
    cfg, cluster, plan, trace = F.config1()
    stages, links = F.load_profiles()
    return engine_cls_or_fn(cfg, F.cluster_with(cluster, links), stages, trace)


def test_reference_engine_reproduces_golden():
    import pipelink

    res = run_with(lambda cfg, cl, st, tr: pipelink.PipelineEngine(cfg, cl, st).run(tr))
    assert res.all_finished
    assert F.digests(res) == GOLD["sha256"]
    assert len(res.decisions) == GOLD["n_decisions"] and res.end_ns == GOLD["end_ns"]


def test_native_scheduler_reproduces_golden():
    from paper_2507_05043_b200.native import NativeScheduler

    def run(cfg, cl, st, tr):
        names = cfg.partition.node_names()
        links = [cl.link(a, b) for a, b in list(zip(names, names[1:])) + [(names[-1], names[0])]]
        sched = NativeScheduler(cfg, st, links, cfg.model.hidden_dim * cfg.model.dtype_bytes)
        try:
            return sched.run(tr, None)
        finally:
            sched.close()

    res = run_with(run)
    assert F.digests(res) == GOLD["sha256"]
