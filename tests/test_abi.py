"""The C-ABI library loads (no GPU needed) and exports every symbol include/b200link.h declares."""

import ctypes
import re
from pathlib import Path

from paper_2507_05043_b200 import _native as N

HEADER = Path(__file__).resolve().parent.parent / "include" / "b200link.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(pl_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(N.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.pl_abi_version() == 1


def test_pure_host_queries():
    lib = N.lib()
    # argmax partials = tiles * T * 8; split-K partials = splits * N * Tp * 4
    assert lib.pl_gemm_workspace_bytes(16, 128256, 4096, N.EPI_ARGMAX) == 1002 * 16 * 8
    assert lib.pl_gemm_workspace_bytes(300, 4096, 4096, N.EPI_NONE) == 0   # prefill: no split-K
    # split counts depend on (N, K) only: L3 o-proj 5 splits; long-K down rounded up to 8
    assert lib.pl_gemm_workspace_bytes(64, 4096, 4096, N.EPI_RESIDUAL) == 5 * 4096 * 64 * 4
    assert lib.pl_gemm_workspace_bytes(64, 4096, 14336, N.EPI_RESIDUAL) == 8 * 4096 * 64 * 4
    assert lib.pl_gemm_workspace_bytes(16, 4096, 14336, N.EPI_RESIDUAL) == 8 * 4096 * 16 * 4
    # decode splits: ceil(pages / 16) per request -- context-length driven only
    assert lib.pl_attn_decode_workspace_bytes(16, 32, 1024, 128) == 0
    assert lib.pl_attn_decode_workspace_bytes(16, 32, 1100, 128) == 2048 + 16 * 32 * 2 * (128 * 4 + 8)
    assert lib.pl_nccl_version() >= 22800


def test_errors_map_to_reference_hierarchy():
    import pytest

    lib = N.lib()
    rc = lib.pl_gemm(None, 0, None, 0, None, None, 0, None, 0, 1, 1, 64, 0, None, 0, None, None)
    assert rc == N.PL_ERR_CONFIG
    with pytest.raises(N.ConfigError):
        N.check(rc, "pl_gemm")
    assert "null operand" in N.last_error()
    uid = (ctypes.c_uint8 * 8)()
    with pytest.raises(N.ConfigError):
        N.call("pl_nccl_unique_id", uid, 8)


def test_packed_weight_entry_points_validate_before_touching_the_gpu():
    import pytest

    lib = N.lib()
    assert lib.pl_pack_weight(None, 64, 256, 64, 0, None, None) == N.PL_ERR_CONFIG
    assert "null argument" in N.last_error()
    rc = lib.pl_gemm_packed(None, 0, None, None, None, 0, None, 0, 1, 256, 64, 0, None, 0, None, None)
    with pytest.raises(N.ConfigError):
        N.check(rc, "pl_gemm_packed")
    assert "null operand" in N.last_error()
