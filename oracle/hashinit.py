"""ORACLE (test infrastructure only): counter-based synthetic initialisation.

Independent numpy restatement of the generator behind ``pl_fill_hash_bf16``
(paper_2507_05043_b200/csrc/kernels.cu) so the CPU oracle and the GPU build
start from bit-identical bf16 weights and prompt token ids.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg import this.

    key  = mix(seed * 0x9E3779B9 + tensor_id * 0x85EBCA6B + 0x632BE5AB)
    key2 = mix(key ^ 0x5bd1e995)
    h    = mix(mix(i + key) ^ key2)                       (uint32 wrap-around)
    w[i] = bf16_rne( f32(int(h >> 8) - 2^23) * f32(scale * 2^-23) + f32(offset) )
"""

from __future__ import annotations

import numpy as np

M32 = np.uint32(0xFFFFFFFF)


def _mix(x: np.ndarray, inplace: bool = False) -> np.ndarray:
    if not inplace:
        x = x.astype(np.uint32, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    return x


def _mix_scalar(x: int) -> int:
    return int(_mix(np.array([x & 0xFFFFFFFF], dtype=np.uint32))[0])


def keys(seed: int, tensor_id: int) -> tuple[int, int]:
    key = _mix_scalar((seed * 0x9E3779B9 + tensor_id * 0x85EBCA6B + 0x632BE5AB) & 0xFFFFFFFF)
    key2 = _mix_scalar(key ^ 0x5BD1E995)
    return key, key2


def hash_u32(n: int, seed: int, tensor_id: int, start: int = 0) -> np.ndarray:
    key, key2 = keys(seed, tensor_id)
    h = np.arange(n, dtype=np.uint32)          # i < 2^32 (tensors are < 2^32 elements)
    with np.errstate(over="ignore"):
        h += np.uint32((start + key) & 0xFFFFFFFF)
        _mix(h, inplace=True)
        h ^= np.uint32(key2)
    return _mix(h, inplace=True)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    with np.errstate(over="ignore"):
        r = (u >> np.uint32(16)) & np.uint32(1)
        r += np.uint32(0x7FFF)
        r += u                                   # finite inputs never wrap
    return (r >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def hash_bf16_bits(n: int, seed: int, tensor_id: int, scale: float, offset: float = 0.0,
                   start: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    out = np.empty(n, dtype=np.uint16)
    mult = np.float32(scale) * np.float32(2.0 ** -23)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        h = hash_u32(m, seed, tensor_id, start + a)
        h >>= np.uint32(8)
        v = h.view(np.int32)
        v -= np.int32(8388608)
        w = v.astype(np.float32)
        w *= mult
        if offset:
            w += np.float32(offset)
        out[a:a + m] = f32_to_bf16_bits(w)
    return out


def hash_tokens(n: int, seed: int, tensor_id: int, vocab: int, start: int = 0) -> np.ndarray:
    """Prompt token ids: hash mod vocab (int64)."""
    return (hash_u32(n, seed, tensor_id, start).astype(np.int64) % vocab).astype(np.int64)


# ------------------------------------------------------------------ torch --
# The same generator restated on torch int64 tensors (uint32 arithmetic kept in the low
# 32 bits; int64 products wrap modulo 2^64, which preserves them), so the oracle can
# build multi-GB weight sets on many host threads -- or on a GPU through torch's own
# elementwise ops, independent of this repo's kernels.  Bit-identical to
# hash_bf16_bits / hash_tokens (tests/test_oracle_hash.py).

_M = 0xFFFFFFFF


def _mix_t(x):
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & _M
    return x ^ (x >> 16)


def hash_u32_torch(n: int, seed: int, tensor_id: int, start: int = 0, device="cpu"):
    import torch

    key, key2 = keys(seed, tensor_id)
    h = torch.arange(n, dtype=torch.int64, device=device)
    h = (h + ((start + key) & _M)) & _M
    h = _mix_t(h) ^ key2
    return _mix_t(h)


def hash_bf16_torch(shape, seed: int, tensor_id: int, scale: float, offset: float = 0.0,
                    device="cpu", chunk: int = 1 << 26):
    """bf16 tensor of `shape` with the bits of hash_bf16_bits (fp32 multiply, then add,
    then round-to-nearest-even to bf16 -- two separate torch ops, never fused)."""
    import torch

    n = int(np.prod(shape))
    mult = float(np.float32(scale) * np.float32(2.0 ** -23))
    off = float(np.float32(offset))
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        h = hash_u32_torch(m, seed, tensor_id, a, device)
        w = ((h >> 8) - 8388608).to(torch.float32) * mult
        if offset:
            w = w + off
        out[a:a + m] = w.to(torch.bfloat16)
    return out.reshape(shape)
