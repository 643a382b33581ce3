"""Decoder shapes and the synthetic-model contract.

``pipelink.ModelSpec`` (placement.py:134-151) carries only what partitioning
and payload sizing need (layers, hidden_dim, dtype_bytes, bytes_per_layer).
The real forward needs heads, FFN width, vocabulary and RoPE/RMSNorm
constants, so they live here in ``DecoderSpec``; ``DecoderSpec.model_spec()``
produces the matching reference ``ModelSpec`` so the engine's payload sizing
(engine.py:294, 406) equals the bf16 residual-stream bytes actually sent.

Weights are synthetic and deterministic: every tensor is filled on the GPU by
the counter-based hash of (seed, tensor_id, element index) (pl_fill_hash_bf16),
so the CPU oracle can regenerate bit-identical values.

Layouts (row-major bf16):
  w_qkv      [(Hq + 2 Hkv) hd, d]   rows = q heads | k heads | v heads
  w_o        [d, Hq hd]
  w_gate_up  [2 ffn, d]             64-row blocks [gate rows j..j+63 | up rows j..j+63]
  w_down     [d, ffn]
  embed, lm_head [vocab, d]         (untied)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from ._pipelink import pipelink

BLOCK_SIZE = 64  # tokens per paged-KV block

# tensor ids for the hash init
T_ATTN_NORM, T_QKV, T_QKV_BIAS, T_O, T_MLP_NORM, T_GATE_UP, T_DOWN = range(7)
T_EMBED = 0xFFFF0001
T_FINAL_NORM = 0xFFFF0002
T_LM_HEAD = 0xFFFF0003
T_PROMPT = 0xFFFF1000  # + request id


def layer_tensor_id(layer: int, kind: int) -> int:
    return (layer << 4) | kind


@dataclass(frozen=True)
class DecoderSpec:
    name: str
    num_layers: int
    d: int
    Hq: int
    Hkv: int
    hd: int
    ffn: int
    vocab: int
    rope_theta: float
    eps: float
    qkv_bias: bool = False
    # init (uniform +-scale; std 0.02 <=> scale 0.02*sqrt(3))
    weight_scale: float = 0.02 * math.sqrt(3.0)
    embed_scale: float = 0.02 * math.sqrt(3.0)
    norm_jitter: float = 0.05
    bias_scale: float = 0.02
    # "peaked" init: embed ~ U(+-peaked_embed_scale), lm_head[v] = lm_alpha * embed[(v+1) % V].
    # The token embedding then dominates the residual stream through all layers
    # (|e|^2 = d*s^2/3 vs max_v <layer contributions, e_v>), so argmax margins dwarf
    # bf16/accumulation-order differences and greedy ids are robustly identical.
    peaked: bool = False
    lm_alpha: float = 4.0
    peaked_embed_scale: float = 8.0

    def __post_init__(self) -> None:
        if self.Hq % self.Hkv:
            raise pipelink.ConfigError("Hq must be a multiple of Hkv")
        if self.hd != 128:
            raise pipelink.ConfigError("head_dim must be 128 (kernel family)")
        if self.d % 64 or self.ffn % 64:
            raise pipelink.ConfigError("d and ffn must be multiples of 64")

    @property
    def qkv_dim(self) -> int:
        return (self.Hq + 2 * self.Hkv) * self.hd

    @property
    def attn_dim(self) -> int:
        return self.Hq * self.hd

    def layer_params(self) -> int:
        p = self.qkv_dim * self.d + self.d * self.attn_dim + 3 * self.ffn * self.d + 2 * self.d
        if self.qkv_bias:
            p += self.qkv_dim
        return p

    def layer_bytes(self) -> int:
        return 2 * self.layer_params()

    def kv_bytes_per_token_layer(self) -> int:
        return 2 * self.Hkv * self.hd * 2

    def model_spec(self) -> "pipelink.ModelSpec":
        return pipelink.ModelSpec(
            name=self.name,
            num_layers=self.num_layers,
            hidden_dim=self.d,
            dtype_bytes=2,
            bytes_per_layer=self.layer_bytes(),
        )

    def with_(self, **kw) -> "DecoderSpec":
        return replace(self, **kw)


TINY = DecoderSpec("tiny-llama", num_layers=4, d=256, Hq=2, Hkv=1, hd=128, ffn=768, vocab=512,
                   rope_theta=1e4, eps=1e-5)
LLAMA3_8B = DecoderSpec("llama3-8b-shape", num_layers=32, d=4096, Hq=32, Hkv=8, hd=128,
                        ffn=14336, vocab=128256, rope_theta=5e5, eps=1e-5)
QWEN2_72B = DecoderSpec("qwen2-72b-shape", num_layers=80, d=8192, Hq=64, Hkv=8, hd=128,
                        ffn=29568, vocab=152064, rope_theta=1e6, eps=1e-6, qkv_bias=True)

PRESETS = {s.name: s for s in (TINY, LLAMA3_8B, QWEN2_72B)}


def rope_table(spec: DecoderSpec, max_pos: int) -> torch.Tensor:
    """bf16 [max_pos, hd] = [cos | sin] of the default (unscaled) RoPE.

    Computed once on the host in fp32 exactly as HF's LlamaRotaryEmbedding
    (modeling_llama.py:111-135): inv_freq = 1 / theta^(2i/hd), angle =
    pos * inv_freq (fp32), cos/sin in fp32, cast to bf16.
    """
    hd = spec.hd
    inv_freq = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    pos = torch.arange(max_pos, dtype=torch.int64).float()
    ang = pos[:, None] * inv_freq[None, :]
    return torch.cat([ang.cos(), ang.sin()], dim=1).to(torch.bfloat16).contiguous()


def prompt_tokens(seed: int, request_id: int, length: int, vocab: int) -> np.ndarray:
    """Synthetic prompt ids: hash(seed, T_PROMPT + request id, position) mod vocab."""
    key = _mix(np.array([(seed * 0x9E3779B9 + (T_PROMPT + request_id) * 0x85EBCA6B + 0x632BE5AB)
                         & 0xFFFFFFFF], dtype=np.uint32))[0]
    key2 = _mix(np.array([int(key) ^ 0x5BD1E995], dtype=np.uint32))[0]
    i = np.arange(length, dtype=np.uint32)
    with np.errstate(over="ignore"):
        h = _mix(_mix(i + key) ^ key2)
    return (h.astype(np.int64) % vocab).astype(np.int64)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint32, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    return x
