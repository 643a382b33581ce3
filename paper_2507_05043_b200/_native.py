"""ctypes binding of libb200link.so (include/b200link.h).

The library is built in-tree by ``paper_2507_05043_b200.build`` and loaded from
``paper_2507_05043_b200/_lib``.  There is no fallback: if the shared library
is missing the import of any compute entry point raises.  Status codes map to
the reference's exception hierarchy (pipelink/errors.py:4-39).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from ._pipelink import pipelink

ConfigError = pipelink.ConfigError
ProtocolError = pipelink.ProtocolError
PipelinkError = pipelink.PipelinkError

LIB_PATH = Path(os.environ.get("PL_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libb200link.so")

PL_OK, PL_ERR_CONFIG, PL_ERR_PROTOCOL, PL_ERR_CUDA = 0, 1, 2, 3
EPI_NONE, EPI_BIAS, EPI_RESIDUAL, EPI_SWIGLU, EPI_ARGMAX = 0, 1, 2, 3, 4

vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float


class LayerWeights(C.Structure):
    _fields_ = [
        ("attn_norm", vp), ("w_qkv", vp), ("b_qkv", vp), ("w_o", vp), ("mlp_norm", vp),
        ("w_gate_up", vp), ("w_down", vp), ("k_cache", vp), ("v_cache", vp),
    ]


class StageConfig(C.Structure):
    _fields_ = [
        ("d", i32), ("Hq", i32), ("Hkv", i32), ("hd", i32), ("ffn", i32), ("num_layers", i32),
        ("vocab", i64), ("eps", f32), ("block_size", i32), ("max_blocks_per_req", i32),
        ("max_pos", i32), ("num_blocks", i64), ("is_first", i32), ("is_last", i32), ("max_tokens", i32),
        ("max_reqs", i32), ("max_ctx", i32), ("embed", vp), ("final_norm", vp), ("lm_head", vp),
        ("cos_sin", vp),
    ]


class MicroBatch(C.Structure):
    _fields_ = [
        ("T", i32), ("R", i32), ("phase", i32), ("max_seqlen", i32), ("max_ctx", i32),
        ("meta", vp), ("token_ids", vp), ("last_token", vp), ("hidden", vp), ("out_ids", vp),
        ("n_decode", i32), ("peer_hidden", vp),
    ]


f64 = C.c_double


class SchedConfig(C.Structure):
    _fields_ = [
        ("n_stages", i32), ("n_links", i32), ("max_batched_tokens", i64), ("max_batch_size", i32),
        ("n_max", i32), ("bubble_epsilon", f64), ("gain_delta", f64), ("fixed_compute", i32),
        ("decision_stride", i32), ("chunk_size", i64), ("fcfs", i32), ("allow_mixed", i32),
        ("bytes_per_token", i64), ("feedback_bytes", i64), ("prof_off", vp), ("prof_x", vp),
        ("prof_y", vp), ("link_latency_s", vp), ("link_bandwidth", vp),
    ]


class PipelineConfig(C.Structure):
    _fields_ = [
        ("n_stages", i32), ("n_slots", i32), ("max_blocks", i32), ("block_size", i32),
        ("num_blocks", i64), ("max_tokens", i32), ("max_reqs", i32), ("d", i32), ("throttle", i32),
        ("record_links", i32), ("stage", vp), ("stream", vp), ("device", vp), ("meta_dev", vp),
        ("ids_dev", vp), ("hidden", vp), ("out_ids", vp), ("comm", vp), ("ids_recv", vp),
        ("fuse_transport", i32),
    ]


_SIGS = {
    "pl_abi_version": (i32, []),
    "pl_preload_kernels": (i32, []),
    "pl_last_error": (C.c_char_p, []),
    "pl_device_sm_count": (i32, [i32]),
    "pl_launch_count": (i64, []),
    "pl_fill_hash_bf16": (i32, [vp, i64, u32, u32, f32, f32, vp]),
    "pl_embed": (i32, [vp, vp, vp, vp, i64, i64, i32, vp, vp]),
    "pl_rmsnorm": (i32, [vp, i64, vp, vp, f32, i64, i32, vp, i64, vp]),
    "pl_gemm_workspace_bytes": (i64, [i64, i64, i64, i32]),
    "pl_gemm": (i32, [vp, i64, vp, i64, vp, vp, i64, vp, i64, i64, i64, i64, i32, vp, i64, vp, vp]),
    "pl_pack_weight": (i32, [vp, i64, i64, i64, i32, vp, vp]),
    "pl_gemm_packed": (i32, [vp, i64, vp, vp, vp, i64, vp, i64, i64, i64, i64, i32, vp, i64, vp, vp]),
    "pl_rope_kv_write": (i32, [vp, i64, vp, vp, vp, i32, vp, vp, i32, i64, i32, i32, i32, vp]),
    "pl_attn_prefill": (i32, [vp, i64, vp, i32, i32, i32, i32, i32, f32, vp, i64, vp]),
    "pl_attn_prefill_ex": (i32, [vp, i64, i64, vp, i32, i32, i32, i32, i32, f32, vp, i64, i32, vp]),
    "pl_attn_decode_workspace_bytes": (i64, [i32, i32, i32, i32]),
    "pl_attn_decode": (i32, [vp, i64, vp, vp, i64, i32, vp, i32, vp, i32, i32, i32, i32, i32, f32, vp, i64, vp, i64, vp]),
    "pl_lmhead_workspace_bytes": (i64, [i32, i64]),
    "pl_lmhead_argmax": (i32, [vp, i64, vp, i64, i32, i32, vp, vp, i64, vp]),
    "pl_token_scatter": (i32, [vp, vp, vp, i32, vp, vp, i32, vp]),
    "pl_stage_workspace_bytes": (i64, [C.POINTER(StageConfig)]),
    "pl_stage_create": (i32, [C.POINTER(StageConfig), C.POINTER(LayerWeights), vp, i64, C.POINTER(vp)]),
    "pl_stage_forward": (i32, [vp, C.POINTER(MicroBatch), vp]),
    "pl_stage_pack_weights": (i32, [vp, vp]),
    "pl_stage_destroy": (i32, [vp]),
    "pl_stage_probe": (i32, [vp, i32]),
    "pl_stage_chain_trace": (i32, [vp, vp, i64, C.POINTER(i32)]),
    "pl_stage_chain_bench": (i32, [vp, i32, i32, i32, vp]),
    "pl_stage_probe_read": (i32, [vp, C.POINTER(f32), C.POINTER(i32), i32, C.POINTER(i32)]),
    "pl_nccl_version": (i32, []),
    "pl_nccl_unique_id": (i32, [C.POINTER(C.c_uint8), i32]),
    "pl_comm_init_rank": (i32, [C.POINTER(C.c_uint8), i32, i32, C.POINTER(vp)]),
    "pl_comm_destroy": (i32, [vp]),
    "pl_p2p_send": (i32, [vp, vp, i64, i32, vp]),
    "pl_p2p_recv": (i32, [vp, vp, i64, i32, vp]),
    "pl_record_globaltimer": (i32, [vp, vp]),
    "pl_gate_until_ns": (i32, [vp, u64, vp]),
    "pl_memcpy_async": (i32, [vp, vp, i64, vp]),
    "pl_enable_peer_access": (i32, [i32, vp]),
    "pl_sched_create": (i32, [C.POINTER(SchedConfig), C.POINTER(vp)]),
    "pl_sched_destroy": (i32, [vp]),
    "pl_sched_choose_n": (i32, [vp, i64, i32, C.POINTER(i32), C.POINTER(i64), C.POINTER(f64)]),
    "pl_sched_run": (i32, [vp, vp, i64, i64, vp]),
    "pl_sched_counts": (i32, [vp, vp]),
    "pl_sched_read": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "pl_pipeline_create": (i32, [C.POINTER(PipelineConfig), C.POINTER(vp)]),
    "pl_pipeline_destroy": (i32, [vp]),
    "pl_pipeline_set_requests": (i32, [vp, i64, vp, vp, vp, vp, i32]),
    "pl_pipeline_counts": (i32, [vp, vp]),
    "pl_pipeline_read": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """The loaded library; raises if it was not built (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise PipelinkError(
                        f"{LIB_PATH} missing: build it with `python -m paper_2507_05043_b200.build`"
                    )
                L = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                if L.pl_abi_version() != 1:
                    raise PipelinkError("libb200link ABI version mismatch")
                _lib = L
    return _lib


def last_error() -> str:
    msg = lib().pl_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == PL_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == PL_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == PL_ERR_PROTOCOL:
        raise ProtocolError(msg)
    raise PipelinkError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
