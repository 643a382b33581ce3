"""Torch-facing wrappers of the libb200link kernel entry points.

Thin: each function checks shapes, allocates outputs/workspaces with torch's
caching allocator and calls one C-ABI function on the current CUDA stream.
Used by the stage executor's setup and by the kernel parity tests; the hot
loop itself goes through ``pl_stage_forward`` (one FFI call per micro-batch).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from ._native import EPI_ARGMAX, EPI_BIAS, EPI_NONE, EPI_RESIDUAL, EPI_SWIGLU  # noqa: F401

BF16 = torch.bfloat16


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream: torch.cuda.Stream | None = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise N.ConfigError("libb200link kernels take CUDA tensors only (no CPU fallback)")


_WS: dict = {}


def _workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """Per-device scratch reused across calls (stream-ordered on the current stream)."""
    buf = _WS.get(device)
    if buf is None or buf.numel() < nbytes:
        # zeroed once: stream-K tile counters must start at 0 (each launch re-zeroes its own)
        buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[device] = buf
    return buf


def fill_hash_(t: torch.Tensor, seed: int, tensor_id: int, scale: float, offset: float = 0.0,
               stream=None) -> torch.Tensor:
    _need_cuda(t)
    assert t.dtype == BF16 and t.is_contiguous()
    N.call("pl_fill_hash_bf16", _ptr(t), t.numel(), seed & 0xFFFFFFFF, tensor_id & 0xFFFFFFFF,
           float(scale), float(offset), _stream(stream))
    return t


def embed(ids: torch.Tensor | None, table: torch.Tensor, T: int | None = None,
          req_slot: torch.Tensor | None = None, last_token: torch.Tensor | None = None,
          out: torch.Tensor | None = None) -> torch.Tensor:
    _need_cuda(ids, table, req_slot, last_token)
    T = ids.numel() if ids is not None else req_slot.numel()
    V, d = table.shape
    out = out if out is not None else torch.empty(T, d, dtype=BF16, device=table.device)
    N.call("pl_embed", _ptr(ids), _ptr(req_slot), _ptr(last_token), _ptr(table), V, T, d, _ptr(out),
           _stream())
    return out


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float, row_idx: torch.Tensor | None = None,
            out: torch.Tensor | None = None) -> torch.Tensor:
    _need_cuda(x, w, row_idx)
    rows = row_idx.numel() if row_idx is not None else x.shape[0]
    d = x.shape[1]
    out = out if out is not None else torch.empty(rows, d, dtype=BF16, device=x.device)
    N.call("pl_rmsnorm", _ptr(x), x.stride(0), _ptr(row_idx), _ptr(w), float(eps), rows, d,
           _ptr(out), out.stride(0), _stream())
    return out


def gemm(x: torch.Tensor, w: torch.Tensor, epilogue: int = EPI_NONE,
         bias: torch.Tensor | None = None, residual: torch.Tensor | None = None,
         out: torch.Tensor | None = None) -> torch.Tensor:
    """C[T, N] = epilogue(x[T, K] . w[N, K]^T) on tcgen05 (SWIGLU -> [T, N/2], ARGMAX -> int64 [T])."""
    _need_cuda(x, w, bias, residual, out)
    T, K = x.shape
    Nw, Kw = w.shape
    if K != Kw:
        raise N.ConfigError(f"gemm: K mismatch {K} vs {Kw}")
    ws_bytes = N.lib().pl_gemm_workspace_bytes(T, Nw, K, epilogue)
    ws = _workspace(x.device, ws_bytes)
    ids = None
    if epilogue == EPI_ARGMAX:
        ids = torch.empty(T, dtype=torch.int64, device=x.device)
    elif out is None:
        n_out = Nw // 2 if epilogue == EPI_SWIGLU else Nw
        out = torch.empty(T, n_out, dtype=BF16, device=x.device)
    N.call("pl_gemm", _ptr(x), x.stride(0), _ptr(w), w.stride(0), _ptr(bias), _ptr(out),
           out.stride(0) if out is not None else 0, _ptr(residual),
           residual.stride(0) if residual is not None else 0, T, Nw, K, epilogue, _ptr(ws), ws_bytes,
           _ptr(ids), _stream())
    return ids if epilogue == EPI_ARGMAX else out


def pack_weight(w: torch.Tensor, interleave: bool = False) -> torch.Tensor:
    """w [N, K] -> the packed, pre-swizzled tile layout of the decode GEMMs (same shape/dtype;
    interleave=True for a gate_up weight used with EPI_SWIGLU)."""
    _need_cuda(w)
    Nw, K = w.shape
    out = torch.empty_like(w)
    N.call("pl_pack_weight", _ptr(w), w.stride(0), Nw, K, int(interleave), _ptr(out), _stream())
    return out


def gemm_packed(x: torch.Tensor, wp: torch.Tensor, epilogue: int = EPI_NONE,
                bias: torch.Tensor | None = None, residual: torch.Tensor | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """gemm() with a weight from pack_weight (interleaved iff epilogue == EPI_SWIGLU)."""
    _need_cuda(x, wp, bias, residual, out)
    T, K = x.shape
    Nw, Kw = wp.shape
    if K != Kw:
        raise N.ConfigError(f"gemm: K mismatch {K} vs {Kw}")
    ws_bytes = N.lib().pl_gemm_workspace_bytes(T, Nw, K, epilogue)
    ws = _workspace(x.device, ws_bytes)
    ids = None
    if epilogue == EPI_ARGMAX:
        ids = torch.empty(T, dtype=torch.int64, device=x.device)
    elif out is None:
        out = torch.empty(T, Nw // 2 if epilogue == EPI_SWIGLU else Nw, dtype=BF16, device=x.device)
    N.call("pl_gemm_packed", _ptr(x), x.stride(0), _ptr(wp), _ptr(bias), _ptr(out),
           out.stride(0) if out is not None else 0, _ptr(residual),
           residual.stride(0) if residual is not None else 0, T, Nw, K, epilogue, _ptr(ws), ws_bytes,
           _ptr(ids), _stream())
    return ids if epilogue == EPI_ARGMAX else out


def rope_kv_write(qkv: torch.Tensor, pos: torch.Tensor, slot: torch.Tensor | None,
                  cos_sin: torch.Tensor, k_cache: torch.Tensor | None, v_cache: torch.Tensor | None,
                  Hq: int, Hkv: int, hd: int, block_size: int = 64) -> None:
    _need_cuda(qkv, pos, slot, cos_sin, k_cache, v_cache)
    N.call("pl_rope_kv_write", _ptr(qkv), qkv.stride(0), _ptr(pos), _ptr(slot), _ptr(cos_sin),
           cos_sin.shape[0], _ptr(k_cache), _ptr(v_cache), block_size, qkv.shape[0], Hq, Hkv, hd,
           _stream())


def attn_prefill(qkv: torch.Tensor, cu_seqlens: torch.Tensor, max_seqlen: int, Hq: int, Hkv: int,
                 hd: int, out: torch.Tensor | None = None, impl: int = 0) -> torch.Tensor:
    """impl: 0 default (tcgen05), 1 mma.sync, 2 tcgen05."""
    _need_cuda(qkv, cu_seqlens)
    T = qkv.shape[0]
    out = out if out is not None else torch.empty(T, Hq * hd, dtype=BF16, device=qkv.device)
    R = cu_seqlens.numel() - 1
    N.call("pl_attn_prefill_ex", _ptr(qkv), qkv.stride(0), T, _ptr(cu_seqlens), R, max_seqlen, Hq, Hkv,
           hd, float(hd ** -0.5), _ptr(out), out.stride(0), impl, _stream())
    return out


def attn_decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                block_table: torch.Tensor, ctx_len: torch.Tensor, max_ctx: int, Hq: int, Hkv: int,
                hd: int, out: torch.Tensor | None = None, block_size: int = 64,
                ws: torch.Tensor | None = None) -> torch.Tensor:
    """q: [R, >= Hq*hd] rows (e.g. the q part of the fused qkv buffer).  `ws`: a zero-
    initialised uint8 workspace reused across calls (sized for the largest call with
    pl_attn_decode_workspace_bytes); default a fresh one per call."""
    _need_cuda(q, k_cache, v_cache, block_table, ctx_len)
    R = ctx_len.numel()
    out = out if out is not None else torch.empty(R, Hq * hd, dtype=BF16, device=q.device)
    if ws is None:
        ws_bytes = N.lib().pl_attn_decode_workspace_bytes(R, Hq, max_ctx, hd)
        ws = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)  # split counters start at 0
    else:
        ws_bytes = ws.numel()
    N.call("pl_attn_decode", _ptr(q), q.stride(0), _ptr(k_cache), _ptr(v_cache), k_cache.shape[0],
           block_size,
           _ptr(block_table), block_table.shape[1], _ptr(ctx_len), R, max_ctx, Hq, Hkv, hd,
           float(hd ** -0.5), _ptr(out), out.stride(0), _ptr(ws), ws_bytes, _stream())
    return out


def lmhead_argmax(h: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    return gemm(h, w, EPI_ARGMAX)


def token_scatter(ids: torch.Tensor, req_slot: torch.Tensor, last_token: torch.Tensor,
                  out_pos: torch.Tensor | None = None, gen_tokens: torch.Tensor | None = None) -> None:
    _need_cuda(ids, req_slot, last_token, out_pos, gen_tokens)
    N.call("pl_token_scatter", _ptr(ids), _ptr(req_slot), _ptr(out_pos), ids.numel(),
           _ptr(last_token), _ptr(gen_tokens), gen_tokens.stride(0) if gen_tokens is not None else 0,
           _stream())
