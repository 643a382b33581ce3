"""B200-native pipeline-parallel serving hot path for MoLink (arXiv 2507.05043).

Drop-in for the reference ``pipelink`` engine: the reference's unchanged API
(partitioning, ``choose_n``, ``admit_and_batch``, ``LinkQueue``) decides the
schedule; this package executes it -- per-stage decoder forwards as hand-written
sm_100a kernels behind the C ABI in ``include/b200link.h``, inter-stage
activations as NCCL P2P over NVLink.
"""

from ._pipelink import pipelink  # noqa: F401  (must precede the modules below)
from .driver import Backend, PipelineDriver
from .spec import LLAMA3_8B, PRESETS, QWEN2_72B, TINY, DecoderSpec

__all__ = ["B200PipelineEngine", "PipelineDriver", "Backend", "DecoderSpec", "TINY", "LLAMA3_8B",
           "QWEN2_72B", "PRESETS"]


def __getattr__(name):
    # GPU-side modules import torch.cuda machinery lazily
    if name == "B200PipelineEngine":
        from .engine import B200PipelineEngine

        return B200PipelineEngine
    raise AttributeError(name)
