"""``--backend b200`` CLI (§8(f)4): the reference's run config and outputs, real compute.

CPU: ``--backend virtual`` goes through the reference's run_simulation and writes the
reference's output files, byte-identical to ``pipelink simulate`` (pkg/tests/test_cli.py
style).  GPU: ``--backend b200`` on the tiny decoder writes the same virtual outputs (the
schedule is the reference engine's) plus b200.json with device-clock metrics."""

import hashlib
import json

import pytest

import pipelink
import pipelink.cli as RC
from paper_2507_05043_b200 import cli

MB = 1 << 20


def write_config(tmp, gpu_count=2):
    nodes = [{"name": f"b200-{i}", "platform": "linux", "gpu_type": "b200", "gpu_count": 1,
              "gpu_mem_bytes": 180 * (1 << 30), "capacity_score": 1.0, "cpu_score": 1.0, "network_score": 1.0}
             for i in range(gpu_count)]
    links = [{"from": a["name"], "to": b["name"], "latency_s": 2e-6, "bandwidth_bps": 9e11}
             for a in nodes for b in nodes if a is not b]
    (tmp / "cluster.json").write_text(json.dumps({"nodes": nodes, "links": links}))
    run = {
        "cluster": "cluster.json",
        "model": {"name": "tiny-llama", "num_layers": 4, "hidden_dim": 256, "dtype_bytes": 2,
                  "bytes_per_layer": 2 * MB},
        "decoder": "tiny-llama",
        "placement": {"gpu_type": "b200", "gpu_count": gpu_count},
        "trace": {"generate": {"rate": 50.0, "duration": 0.2, "seed": 7}},
        "filter": {"max_input": 128, "max_output": 16},
        "profiles": {"synthetic": {"per_layer_token_cost": 1e-6, "overhead_s": 0.0005}},
        "engine": {"chunk_size": 4096, "scheduling_policy": "decode_priority", "seed": 7},
        "controller": {"max_batched_tokens": 512, "max_batch_size": 16},
    }
    (tmp / "run.json").write_text(json.dumps(run))
    return tmp / "run.json"


def digest(d):
    return {f: hashlib.sha256((d / f).read_bytes()).hexdigest()
            for f in ("report.json", "events.csv", "transport.csv", "decisions.csv")}


def test_virtual_backend_matches_reference_cli(tmp_path):
    cfg = write_config(tmp_path)
    assert cli.main(["simulate", "--config", str(cfg), "--out", str(tmp_path / "a"), "--backend", "virtual"]) == 0
    assert RC.main(["simulate", "--config", str(cfg), "--out", str(tmp_path / "b")]) == 0
    assert digest(tmp_path / "a") == digest(tmp_path / "b")


@pytest.mark.gpu
def test_b200_backend_same_schedule_outputs(tmp_path):
    cfg = write_config(tmp_path)
    assert cli.main(["simulate", "--config", str(cfg), "--out", str(tmp_path / "g")]) == 0
    assert RC.main(["simulate", "--config", str(cfg), "--out", str(tmp_path / "r")]) == 0
    assert digest(tmp_path / "g") == digest(tmp_path / "r")
    b = json.loads((tmp_path / "g" / "b200.json").read_text())
    assert b["device_tok_s"] > 0 and b["tokens"]
