"""In-tree build of libfcg.so (nvcc, sm_100a).

The shared library is built next to the package so it travels with the repo
snapshot to the GPU box; no JIT cache is involved.  Objects go to build/.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "fcg"
LIB = PKG / "libfcg.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "--std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libfcg.so")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) \
        + [ROOT / "include" / "fcg.h", Path(__file__)]


def _extra_flags() -> list:
    return os.environ.get("FCG_NVCC_EXTRA", "").split()  # diagnostic A/B builds


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    stamp = BUILD / "flags.txt"  # a build with other flags is stale, whatever the mtimes say
    if (stamp.read_text() if stamp.exists() else "") != " ".join(_extra_flags()):
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    nvcc = _nvcc()
    BUILD.mkdir(parents=True, exist_ok=True)
    logs = {}

    def compile_one(src: Path):
        obj = BUILD / (src.stem + ".o")
        extra = _extra_flags()
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs[src.name] = res.stdout + res.stderr
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    (BUILD / "flags.txt").write_text(" ".join(_extra_flags()))
    (BUILD / "ptxas.log").write_text("\n".join(f"== {k}\n{v}" for k, v in sorted(logs.items())))
    if verbose:
        print((BUILD / "ptxas.log").read_text())
    return LIB


if __name__ == "__main__":
    import sys
    build_library(force="-f" in sys.argv, verbose=True)
    print(LIB)
