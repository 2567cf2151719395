"""Build libgo_b200.so in-tree with nvcc for sm_100a (no torch JIT, no CMake).

    python -m paper_2010_12438_b200.build          # incremental
    python -m paper_2010_12438_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "build_obj"
LIB = PKG / "libgo_b200.so"
INCLUDE = PKG.parent / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
          "--expt-relaxed-constexpr", "-I", str(INCLUDE), "-I", str(CSRC)]
# float64 paths that must be bit-exact with the reference: no FMA contraction
EXACT = {"des.cu", "sample.cu", "graph.cu"}


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers_mtime():
    hs = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, force: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    if (not force and obj.exists() and obj.stat().st_mtime >= src.stat().st_mtime
            and obj.stat().st_mtime >= _headers_mtime()):
        return obj
    flags = list(COMMON)
    if src.name in EXACT:
        flags += ["-fmad=false"]
    cmd = [NVCC, *ARCH, *flags, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if (force or not LIB.exists()
            or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs)):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    _build_probe(force)
    if verbose:
        print("built", LIB)
    return LIB


PROBE_SRC = PKG.parent / "scripts" / "mufu_peak.cu"
PROBE = PKG.parent / "scripts" / "mufu_peak"


def _build_probe(force: bool) -> None:
    """The MUFU/FMA throughput probe bench.py uses as the exp2 roofline denominator."""
    if not PROBE_SRC.exists():
        return
    if not force and PROBE.exists() and PROBE.stat().st_mtime >= PROBE_SRC.stat().st_mtime:
        return
    cmd = [NVCC, *ARCH, "-O3", "-o", str(PROBE), str(PROBE_SRC)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {PROBE_SRC.name}:\n{res.stderr}")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
