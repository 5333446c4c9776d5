"""Double-precision host I/O of the C ABI (pald_gpu_cohesion_f64io*,
csrc/pald_hostio.cu): the calls the C++ shim makes for the reference's own
types (DistanceMatrix doubles in, PaldResult double C out; types.hpp:43-119,
to_real<float> blocked.hpp:91-96, collect_result blocked.hpp:352-359). The
conversions are pipelined with the banded transfers (rows converted just
before their H2D copy, C widened as its D2H bands land), so the results must
equal the plain fp32 call on the converted matrix bit for bit, on the banded
(n > 2048) and the whole-matrix path, for begin/outputs/end in any order."""
import ctypes as C

import numpy as np
import pytest

from helpers import int_upper, random_upper

pytestmark = pytest.mark.gpu


def _f32(lib, _lib, d32, alg, flags=0):
    n = d32.shape[0]
    o = _lib.make_opts(algorithm=alg, flags=flags)
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    assert lib.pald_gpu_cohesion_f32(d32.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, None) == 0
    return u, c


@pytest.mark.parametrize("n,kind", [(300, "rand"), (700, "ties"), (2304, "rand"), (4200, "rand")])
@pytest.mark.parametrize("mode", ["one_call", "outputs_early", "outputs_at_end"])
def test_f64io_matches_f32_call(n, kind, mode):
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    d = (random_upper(n, 11) if kind == "rand" else int_upper(n, 12)).astype(np.float64)
    # doubles that are not representable in fp32: the conversion is to_real<float>
    d = np.where(d > 0, d * (1.0 + 2.0 ** -30), 0.0)
    d = np.maximum(d, d.T)
    d32 = d.astype(np.float32)
    u_ref, c_ref = _f32(lib, _lib, d32, _lib.PAIRWISE)
    o = _lib.make_opts(algorithm=_lib.PAIRWISE)
    u = np.full((n, n), -1, np.int32)
    c = np.full((n, n), np.nan, np.float64)
    pt = _lib.PhaseTimes()
    if mode == "one_call":
        rc = lib.pald_gpu_cohesion_f64io(d.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, C.byref(pt))
    else:
        job = C.c_void_p()
        assert lib.pald_gpu_cohesion_f64io_begin(d.ctypes.data, n, C.byref(o), C.byref(job)) == 0
        if mode == "outputs_early":
            assert lib.pald_gpu_cohesion_f64io_outputs(job, u.ctypes.data, c.ctypes.data) == 0
            assert lib.pald_gpu_cohesion_f64io_outputs(job, u.ctypes.data, c.ctypes.data) == _lib.ERR_VALIDATION
            rc = lib.pald_gpu_cohesion_f64io_end(job, None, None, C.byref(pt))
        else:
            rc = lib.pald_gpu_cohesion_f64io_end(job, u.ctypes.data, c.ctypes.data, C.byref(pt))
    assert rc == 0, _lib.last_error()
    assert np.array_equal(u, u_ref)
    assert np.array_equal(c, c_ref.astype(np.float64))  # widened, bit for bit
    assert pt.total_seconds > 0 and pt.total_seconds < 60
    assert pt.overhead_seconds >= 0 and pt.focus_seconds > 0 and pt.cohesion_seconds > 0


def test_f64io_triplet_accurate_and_null_u():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    n = 2500
    d = random_upper(n, 5).astype(np.float64)
    u_ref, c_ref = _f32(lib, _lib, d.astype(np.float32), _lib.TRIPLET, _lib.FLAG_ACCURATE)
    o = _lib.make_opts(algorithm=_lib.TRIPLET, flags=_lib.FLAG_ACCURATE)
    c = np.empty((n, n), np.float64)
    assert lib.pald_gpu_cohesion_f64io(d.ctypes.data, n, C.byref(o), None, c.ctypes.data, None) == 0
    assert np.array_equal(c, c_ref.astype(np.float64))


def test_f64io_errors_leave_the_library_usable():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    n = 2100
    d = random_upper(n, 6).astype(np.float64)
    bad = d.copy()
    bad[5, 1700] = -1.0  # found on the device, in a late band
    bad[1700, 5] = -1.0
    o = _lib.make_opts(algorithm=_lib.PAIRWISE)
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float64)
    job = C.c_void_p()
    assert lib.pald_gpu_cohesion_f64io_begin(bad.ctypes.data, n, C.byref(o), C.byref(job)) == 0
    assert lib.pald_gpu_cohesion_f64io_outputs(job, u.ctypes.data, c.ctypes.data) == 0
    assert lib.pald_gpu_cohesion_f64io_end(job, None, None, None) == _lib.ERR_VALIDATION
    assert "must be positive" in _lib.last_error()
    # end() without any output pointer: refused, the job is still cleaned up
    job = C.c_void_p()
    assert lib.pald_gpu_cohesion_f64io_begin(d.ctypes.data, n, C.byref(o), C.byref(job)) == 0
    assert lib.pald_gpu_cohesion_f64io_end(job, None, None, None) == _lib.ERR_VALIDATION
    # and the next call works
    assert lib.pald_gpu_cohesion_f64io(d.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, None) == 0
    u_ref, c_ref = _f32(lib, _lib, d.astype(np.float32), _lib.PAIRWISE)
    assert np.array_equal(u, u_ref) and np.array_equal(c, c_ref.astype(np.float64))
    assert lib.pald_gpu_release_host_staging() == 0


def test_host_prefault_zeroes():
    from paper_2307_16652_b200 import _lib

    lib = _lib.load()
    a = np.full(5_000_003, 7, np.uint8)
    assert lib.pald_gpu_host_prefault(a.ctypes.data, a.size) == 0
    assert not a.any()
    assert lib.pald_gpu_host_prefault(None, 0) == 0
