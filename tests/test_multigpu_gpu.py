"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise).

Each check runs under torchrun, one rank per GPU, with NCCL P2P between ranks:
* scripts/check_multigpu.py -- virtual-clock engine, stages split over ranks:
  schedule == pipelink's, greedy ids == CPU oracle;
* scripts/check_live.py -- live 2-stage NVLink pipeline (run_device_demo):
  token counts == the virtual run's, ids == CPU oracle;
* 8 stages on 4 GPUs in one process (two stages per GPU, never two processes on
  one GPU -- spinning NCCL kernels of co-resident processes can deadlock).
"""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(script, *args, nproc=2, timeout=600, gpus=None, env=None):
    gpus = gpus or nproc
    if torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "scripts" / script),
           *args]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, "PYTHONPATH": str(ROOT), **(env or {})})
    assert p.returncode == 0, p.stdout[-20000:] + p.stderr[-4000:]
    return p.stdout


def test_two_ranks_two_stages_tiny():
    out = torchrun("check_multigpu.py")
    assert "8/8 requests identical" in out


def test_two_ranks_four_stages_llama3_width():
    out = torchrun("check_multigpu.py", "--stages", "4", "--model", "l3-2", "--requests", "4",
                   "--prompt", "96", "--decode", "6")
    assert "4/4 requests identical" in out


def test_live_nvlink_pipeline_token_parity():
    out = torchrun("check_live.py")
    assert "token counts == virtual" in out and "20/20 requests identical" in out
    upd = int(out.split("monitor: ")[1].split(" profile updates")[0])
    assert upd >= 2, out  # runtime monitoring replaced the startup profiles while serving


def test_live_nvlink_pipeline_four_stages():
    out = torchrun("check_live.py", nproc=4)
    assert "live 4-stage" in out and "token counts == virtual" in out and "20/20 requests identical" in out


def test_eight_stages_on_four_gpus_one_process():
    """The 8-stage pipeline (the north-star depth) on a 4-GPU box in ONE process, two
    stages per GPU, hops as NVLink peer copies or fused epilogue stores (no two
    processes ever share a GPU): schedule == pipelink's, greedy ids == the oracle."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    import numpy as np

    import pipelink
    from oracle import decoder as OD
    from paper_2507_05043_b200 import LLAMA3_8B, deploy
    from paper_2507_05043_b200.engine import B200PipelineEngine, schedule_key
    from paper_2507_05043_b200.spec import prompt_tokens

    spec = LLAMA3_8B.with_(num_layers=8, peaked=True)
    S = 8
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    cfg = deploy.engine_config(plan, spec, pipelink.ControllerConfig(max_batched_tokens=512, max_batch_size=4))
    trace = deploy.uniform_trace(4, 64, 5)
    prof = [pipelink.synth_profile(hi - lo, 1e-6, 2e-5, stage_id=i) for i, (_, (lo, hi)) in enumerate(plan.stages)]
    eng = B200PipelineEngine(cfg, cluster, prof, decoder=spec, devices=[torch.device("cuda", g) for g in range(4)])
    res = eng.run(trace)
    assert schedule_key(res) == schedule_key(pipelink.PipelineEngine(cfg, cluster, prof).run(trace))
    model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=128)
    want, _ = model.greedy([torch.from_numpy(prompt_tokens(0, r.id, r.input_len, spec.vocab))
                            for r in trace.requests], 5)
    for i, r in enumerate(trace.requests):
        assert np.array_equal(res.b200.tokens[r.id], want[i].numpy())
    eng.close()
