"""Build the sm_100a C-ABI library in-tree (paper_2503_12668_b200/_lib/).

nvcc cross-compiles for B200 without a GPU; the resulting .so travels to the
GPU box with the repo snapshot.  Host code is compiled with
-ffp-contract=off so the host restatement of the RNG (zo2_host_*) performs
the same IEEE operations as the device code.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIBNAME = "libzo2b200.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["zo2_elementwise.cu", "zo2_k2.cu", "zo2_layers.cu", "zo2_gemm_sm100.cu", "zo2_attention.cu",
           "zo2_f64.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("ZO2_NVCC_EXTRA", "").split()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-I", str(INCLUDE), "-I", str(CSRC)]


def lib_path() -> Path:
    return LIBDIR / LIBNAME


def _deps(src: Path) -> list[Path]:
    return [src] + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "zo2b200.h"]


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _compile(src: str, verbose: bool) -> Path:
    s = CSRC / src
    o = LIBDIR / (s.stem + ".o")
    if _stale(o, _deps(s)):
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(s), "-o", str(o)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return o


def build_library(verbose: bool = False) -> Path:
    LIBDIR.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    out = lib_path()
    if _stale(out, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart_static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build_library(verbose=True))
