"""Builds libgolp_b200.so in-tree with nvcc for sm_100a (no torch involved).

    python -m paper_2601_19911_b200.csrc.build        # or __graft_entry__.build()
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
LIB = PKG / "libgolp_b200.so"
SOURCES = ["api.cu", "host_engine.cpp", "runtime.cpp"]
HEADERS = ["common.cuh", "sortnet.cuh", "topk.cuh", "sort.cuh", "join.cuh", "runtime.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-pthread",
    "-Xptxas", "-v",
    "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 path cannot be built")


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [HERE / s for s in SOURCES + HEADERS] + [ROOT / "include" / "golp_b200.h"]
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile libgolp_b200.so (or a tuning variant with extra -D defines at `out`)."""
    target = Path(out).resolve() if out is not None else LIB
    if not force and out is None and not defines and not _stale():
        return LIB
    nvcc = _nvcc()
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-shared", "-o", str(tmp),
           *[str(HERE / s) for s in SOURCES], "-lpthread"]
    proc = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    log = PKG / "build_ptxas.log"
    log.write_text(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}")
    os.replace(tmp, target)
    if verbose:
        sys.stdout.write(proc.stderr)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
