"""C ABI checks that need no GPU: the sm_100a library builds/loads, exports
every entry point include/pald_gpu.h declares, and validates arguments with
the reference's error codes before touching the device."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pald_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pald_gpu_\w+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for s in ("pald_gpu_cohesion_f32", "pald_gpu_cohesion_f32_device", "pald_gpu_plan_focus_counts",
              "pald_gpu_plan_focus_finish", "pald_gpu_plan_cohesion", "pald_gpu_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_lib.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (pald_gpu_\w+)", out.stdout))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_only():
    from paper_2307_16652_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert all("sm_100a" in line for line in out.stdout.splitlines() if "sm_" in line)


def test_abi_version_and_opts_layout():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    assert lib.pald_gpu_abi_version() == 4
    o = _lib.make_opts()
    # v3 prefix (48 bytes) + num_devices + devices[8] + two exchange fields
    assert o.struct_size == C.sizeof(_lib.Opts) == 96  # 48 + 4 + 32 + 8, padded to 8
    assert o.block == o.block_focus == o.block_cohesion == 128 and o.device == -1
    assert o.num_devices == 0 and o.exchange_focus == o.exchange_cohesion == _lib.EXCHANGE_AUTO
    assert _lib.OPTS_V3_SIZE == 48
    assert C.sizeof(_lib.Buffers) == 72 and C.sizeof(_lib.PlanInfo) == 40


def test_v3_sized_options_are_accepted():
    """A caller built against ABI v3 passes the 48-byte struct: it is read
    as one device (argument errors still come back first, no GPU needed)."""
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    d = (C.c_float * 9)()
    c = (C.c_float * 9)()
    o = _lib.make_opts(block=0)
    o.struct_size = _lib.OPTS_V3_SIZE
    o.num_devices = 99  # beyond the v3 prefix: must be ignored
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), None, c, None) == _lib.ERR_VALIDATION
    assert "block size" in _lib.last_error()


def test_device_list_validation():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    d = (C.c_float * 9)()
    c = (C.c_float * 9)()
    o = _lib.make_opts()
    o.num_devices = 9
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), None, c, None) == _lib.ERR_VALIDATION
    assert "num_devices" in _lib.last_error()
    o = _lib.make_opts(exchange_focus=7)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), None, c, None) == _lib.ERR_VALIDATION
    o = _lib.make_opts(exchange_cohesion=_lib.EXCHANGE_RED)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), None, c, None) == _lib.ERR_VALIDATION
    assert "pass 1 only" in _lib.last_error()
    o = _lib.make_opts(devices=[0, 64])  # not a visible device (none are, without a GPU)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), None, c, None) == _lib.ERR_VALIDATION
    assert "not a visible device" in _lib.last_error()


def test_argument_validation_before_device_work():
    """Reference error semantics (blocked.hpp:372, :429-431): ValidationError
    for block sizes < 1, UnsupportedPolicyError for triplet + split --
    checked before any CUDA call, so they hold without a GPU."""
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    d = (C.c_float * 9)()
    u = (C.c_int32 * 9)()
    c = (C.c_float * 9)()
    o = _lib.make_opts(block=0)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), u, c, None) == _lib.ERR_VALIDATION
    assert "block size" in _lib.last_error()
    o = _lib.make_opts(algorithm=_lib.TRIPLET, policy=_lib.INCLUSIVE_SPLIT)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), u, c, None) == _lib.ERR_UNSUPPORTED
    o = _lib.make_opts(algorithm=_lib.TRIPLET, block_focus=0)
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), u, c, None) == _lib.ERR_VALIDATION
    o = _lib.make_opts()
    assert lib.pald_gpu_cohesion_f32(d, 1, C.byref(o), u, c, None) == _lib.ERR_VALIDATION
    o.struct_size = 7
    assert lib.pald_gpu_cohesion_f32(d, 3, C.byref(o), u, c, None) == _lib.ERR_VALIDATION


def test_build_tracks_every_csrc_file():
    """A stale library must rebuild when any kernel header changes (the
    pair-kernel header once escaped the staleness check)."""
    from paper_2307_16652_b200 import _build

    names = {p.name for p in _build.deps()}
    for f in ("pald_gpu.cu", "pald_kernels.cuh", "pald_sym.cuh", "pald_multi.cuh", "pald_internal.h", "pald_gpu.h"):
        assert f in names, f
