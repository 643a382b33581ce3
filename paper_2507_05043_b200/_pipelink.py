"""Locate the reference's unchanged ``pipelink`` package.

The drop-in keeps the reference's Python API (``pkg/src/pipelink``) unchanged:
partitioning, the dynamic micro-batch controller (``choose_n``), continuous
batching (``admit_and_batch``) and the chunked decode-priority ``LinkQueue``
are imported, never re-implemented.  Search order:

1. an already-importable ``pipelink`` (installed, or on ``PYTHONPATH``);
2. ``<repo>/baseline/_ref`` -- the unmodified reference installed with
   ``pip install --target baseline/_ref`` (git-ignored, travels with gpurun);
3. ``/root/reference/pkg/src`` (the read-only reference checkout, dev box only).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

_ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (_ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def ensure_pipelink():
    try:
        return importlib.import_module("pipelink")
    except ImportError:
        pass
    for cand in _CANDIDATES:
        if (cand / "pipelink" / "__init__.py").exists():
            sys.path.insert(0, str(cand))
            return importlib.import_module("pipelink")
    raise ImportError(
        "pipelink (the reference scheduler API) is not importable; install it with "
        "`python -m pip install --no-index --no-build-isolation --target baseline/_ref "
        "<copy of /root/reference/pkg>` or run __graft_entry__.build()"
    )


pipelink = ensure_pipelink()
