"""Committed 8-stage B200 runs replayed through the unmodified reference engine (CPU).

Each ``profiles/r2/multigpu/*s8*.log`` line written by ``scripts/run_stages.py``
carries the stage and link profiles the run measured and the decisions / virtual
span it executed on the GPUs.  ``pipelink.PipelineEngine`` fed the same profiles
must reproduce both exactly — including the run where the reference controller
settled on n = 7 and the virtual span doubled, which is therefore
the reference algorithm's behaviour, not this engine's.
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "scripts"))

LOGS = ["final5_s8_g4.log", "final5_s8_g4_rep2.log", "s8_profiles_rep1.log"]


@pytest.mark.parametrize("name", LOGS)
def test_device_schedule_replays_on_reference(name):
    import controller_bimodal as CB

    out = CB.run(ROOT / "profiles" / "r2" / "multigpu" / name)
    dev, ref = out["device_run"], out["reference_cpu"]
    assert {int(k): v for k, v in dev["decisions"].items()} == ref["decisions"]
    assert dev["virtual_span_s"] == ref["virtual_span_s"]


def test_bimodal_outcome_is_in_the_decode_tables():
    """The n = 7 run's span is ~2x the n = 6 run's on the reference engine itself."""
    import controller_bimodal as CB

    slow = CB.run(ROOT / "profiles" / "r2" / "multigpu" / "final5_s8_g4.log")["reference_cpu"]
    fast = CB.run(ROOT / "profiles" / "r2" / "multigpu" / "final5_s8_g4_rep2.log")["reference_cpu"]
    assert max(slow["decisions"], key=slow["decisions"].get) == 7
    assert max(fast["decisions"], key=fast["decisions"].get) == 6
    assert slow["virtual_span_s"] > 1.8 * fast["virtual_span_s"]
