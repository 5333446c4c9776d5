"""Builds tests/cpp/test_shim.cpp against include/pald_gpu.hpp and the C ABI
library, in both type modes (stand-alone types; the reference's own
pald/types.hpp when /root/reference is present), and runs it."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")


def _build(tmp: Path, ref_types: bool) -> Path:
    from paper_2307_16652_b200._build import LIB_PATH, build

    build()
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    exe = tmp / ("test_shim_ref" if ref_types else "test_shim")
    cmd = ["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "cpp" / "test_shim.cpp"), "-o", str(exe),
           str(LIB_PATH), str(ROOT / "oracle" / "liboracle.so"),
           f"-Wl,-rpath,{LIB_PATH.parent}:{ROOT / 'oracle'}", "-pthread"]
    if ref_types:
        cmd[3:3] = ["-DPALD_GPU_USE_REFERENCE_TYPES", "-I", str(REF_INC)]
    subprocess.run(cmd, check=True)
    return exe


def build_shim_test(tmp: Path, ref_types: bool = False) -> Path:
    """The shim test binary (tests/cpp/test_shim.cpp), for other test modules."""
    return _build(tmp, ref_types)


def test_shim_validation_cpu(tmp_path):
    exe = _build(tmp_path, False)
    out = subprocess.run([str(exe), "--cpu-only"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present")
def test_shim_with_reference_types_cpu(tmp_path):
    exe = _build(tmp_path, True)
    out = subprocess.run([str(exe), "--cpu-only"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_shim_gpu(tmp_path):
    exe = _build(tmp_path, False)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
