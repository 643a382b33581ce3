"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise).

Each check runs under torchrun, one rank per GPU, with NCCL P2P between ranks:
* scripts/check_multigpu.py -- virtual-clock engine, stages split over ranks:
  schedule == pipelink's, greedy ids == CPU oracle;
* scripts/check_live.py -- live 2-stage NVLink pipeline (run_device_demo):
  token counts == the virtual run's, ids == CPU oracle.
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
    assert p.returncode == 0, p.stdout[-6000:] + p.stderr[-2000:]
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


def test_live_nvlink_pipeline_four_stages():
    out = torchrun("check_live.py", nproc=4)
    assert "live 4-stage" in out and "token counts == virtual" in out and "20/20 requests identical" in out


def test_eight_ranks_eight_stages_on_four_gpus():
    """The 8-stage, 8-rank pipeline (the driver's N = 8 shape) on a 4-GPU box, two ranks
    per GPU: schedule == pipelink's on every rank, greedy ids == the CPU oracle."""
    out = torchrun("check_multigpu.py", "--stages", "8", "--model", "l3-2", "--requests", "4",
                   "--prompt", "64", "--decode", "5", nproc=8, gpus=4, env={"PL_OVERSUBSCRIBE_GPUS": "4"})
    assert "world 8, 8 stages: 4/4 requests identical" in out
