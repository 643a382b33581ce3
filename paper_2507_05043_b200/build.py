"""Build libb200link.so in-tree with nvcc for sm_100a.

    python -m paper_2507_05043_b200.build [--force] [-v]

Each ``csrc/*.cu`` compiles to ``_build/*.o`` (incremental on mtime), then one
shared library links against the NCCL that torch ships (pip ``nvidia-nccl-cu12``
2.28.x) so the process holds a single NCCL.  The CUDA runtime is linked
statically (nvcc default), so the library only needs the driver at run time.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
import os as _os

# experiment builds (never the product): PL_BUILD_VARIANT=<name> + PL_NVCC_EXTRA="-D..." build
# into _build_<name>/ and _lib_<name>/, loaded with PL_LIB_PATH=<that .so>
_VARIANT = _os.environ.get("PL_BUILD_VARIANT", "")
OBJ = PKG / ("_build" + (f"_{_VARIANT}" if _VARIANT else ""))
LIB_DIR = PKG / ("_lib" + (f"_{_VARIANT}" if _VARIANT else ""))
LIB = LIB_DIR / "libb200link.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs() -> tuple[Path, Path]:
    import nvidia.nccl  # the NCCL torch loads

    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def _nvcc() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        raise RuntimeError("nvcc not found")
    return nvcc


def _flags() -> list[str]:
    inc, _ = _nccl_dirs()
    return [
        *ARCH,
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC,-fvisibility=hidden,-ffp-contract=off",
        "--expt-relaxed-constexpr",
        f"-I{ROOT / 'include'}",
        f"-I{inc}",
        *_os.environ.get("PL_NVCC_EXTRA", "").split(),
    ]


def _needs(src: Path, obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *deps])


def build(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    OBJ.mkdir(exist_ok=True)
    LIB_DIR.mkdir(exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "b200link.h"]
    flags = _flags()
    jobs = []
    for src in sources:
        obj = OBJ / (src.stem + ".o")
        if force or _needs(src, obj, headers):
            jobs.append(([nvcc, *flags, "-Xptxas", "-v" if verbose else "-O3", "-c", str(src), "-o", str(obj)], src))

    def run(job):
        cmd, src = job
        p = subprocess.run(cmd, capture_output=True, text=True)
        return src, p

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            for src, p in ex.map(run, jobs):
                if verbose and p.stderr:
                    print(p.stderr, file=sys.stderr)
                if p.returncode != 0:
                    raise RuntimeError(f"nvcc failed on {src.name}:\n{p.stdout}\n{p.stderr}")
    objs = [OBJ / (s.stem + ".o") for s in sources]
    if force or jobs or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        _, nccl_lib = _nccl_dirs()
        cmd = [
            nvcc,
            *ARCH,
            "-shared",
            "-o",
            str(LIB),
            *map(str, objs),
            f"-L{nccl_lib}",
            "-l:libnccl.so.2",
            f"-Xlinker=-rpath={nccl_lib}",
        ]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
