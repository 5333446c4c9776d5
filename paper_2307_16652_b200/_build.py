"""In-tree build of the sm_100a C-ABI library (libpald_gpu.so).

The library is compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
only (no PTX fallback, no other architectures) and lands next to this file in
``lib/`` so that the gpurun snapshot carries it to the B200 box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_DIR = PKG_DIR / "lib"
LIB_PATH = LIB_DIR / "libpald_gpu.so"
INCLUDE = PKG_DIR.parent / "include"

SOURCES = [CSRC / "pald_gpu.cu", CSRC / "pald_epilogue.cu", CSRC / "pald_io.cu", CSRC / "pald_hostio.cu"]
def deps() -> list[Path]:
    """Every file the library is built from (sources, kernel headers, ABI)."""
    return sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), *INCLUDE.glob("*.h")])

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-Xlinker", "-soname=libpald_gpu.so",
    "-Xptxas", "-v",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the sm_100a library cannot be built")


def needs_build() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libpald_gpu.so if missing or stale; returns its path."""
    if not force and not needs_build():
        return LIB_PATH
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *NVCC_FLAGS, "-I", str(INCLUDE), "-o", str(tmp), *map(str, SOURCES)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    (LIB_DIR / "ptxas.log").write_text(proc.stdout + proc.stderr)
    os.replace(tmp, LIB_PATH)
    if verbose:
        print(proc.stderr)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True))
