"""Builds the sm_100a C-ABI library ``libmosaic_b200.so`` in-tree with nvcc.

The library is a plain shared object (no torch types in its interface); the
Python host loads it with ctypes. Building in-tree keeps the .so inside the
repository snapshot that travels to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
BUILD = REPO / "build" / "obj"
LIB = PKG_DIR / "libmosaic_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def source_hash(names: tuple[str, ...] | None = None) -> str:
    """sha256 (16 hex digits) of kernel sources -- ``names`` inside csrc/, or
    every csrc/ file plus the C-ABI header -- and the nvcc flags. Evidence
    recorded from a profiler capture (profiles/k3_traffic.json) carries the hash
    of the code it measured; bench.py reports it only while the hash matches."""
    import hashlib

    files = ([CSRC / n for n in names] if names else sorted(CSRC.glob("*")) + [REPO / "include" / "mosaic_b200.h"])
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


K3_SOURCES = ("lmhead.cu", "common.cuh")


def _stale(objs: list[Path]) -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [REPO / "include" / "mosaic_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def _extra_defines() -> list[str]:
    """Experiment-only compile-time knobs, e.g. MOSAIC_NVCC_DEFINES="MOSAIC_K3_STAGES2=7"."""
    return [f"-D{d}" for d in os.environ.get("MOSAIC_NVCC_DEFINES", "").split() if d]


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = sources()
    objs = [BUILD / (s.stem + ".o") for s in srcs]
    if not force and not _stale(objs):
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(pair):
        src, obj = pair
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *_extra_defines(), "-I", str(REPO / "include"), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        return src.name, r.stderr

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        logs = list(ex.map(compile_one, zip(srcs, objs)))
    if verbose:
        for name, log in logs:
            print(f"--- {name}\n{log}", file=sys.stderr)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
