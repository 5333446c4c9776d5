"""Several devices in ONE C-ABI call (pald_gpu_opts.devices, ABI v4;
csrc/pald_multi.cuh): the GPU counterpart of parallel_pairwise /
parallel_triplet's worker count (parallel.hpp:159-222, :257-320).

Only one B200 is available here, so the device list repeats device 0:
every listed "device" gets its own plan, streams and host thread, the
shares of pass 1 / pass 2 are split exactly as on distinct GPUs, and the
exchange kernels read and write the other plans' buffers through the same
pointers they would use over NVLink (a repeated device needs no P2P
enable). The contract under test: U and C bit-identical to one device, for
every transport that runs on one GPU and every pass-2 kernel choice.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from helpers import int_upper, random_upper

pytestmark = pytest.mark.gpu


def host_call(d, algorithm="pairwise", devices=None, policy="strict", xf=0, xc=0, flags=0):
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for

    lib = _lib.load()
    alg = {"pairwise": _lib.PAIRWISE, "triplet": _lib.TRIPLET}[algorithm]
    pol = {"strict": _lib.STRICT, "split": _lib.INCLUSIVE_SPLIT}[policy]
    o = _lib.make_opts(algorithm=alg, policy=pol, devices=devices, exchange_focus=xf, exchange_cohesion=xc,
                       flags=flags)
    n = d.shape[0]
    u = np.full((n, n), -7, np.int32)
    c = np.full((n, n), np.nan, np.float32)
    pt = _lib.PhaseTimes()
    _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, C.byref(pt)))
    assert pt.total_seconds > 0
    return u, c


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


@pytest.mark.parametrize("ndev", [2, 3, 8])
def test_repeated_device_pairwise_pair_kernel(ndev):
    """Random D, n = 2304: pair kernel with tie marks; 3 and 8 shares do not
    divide the 171 tile pairs / the 18 tile rows evenly."""
    d = random_upper(2304, 8)
    u1, c1 = host_call(d)
    u, c = host_call(d, devices=[0] * ndev)
    assert np.array_equal(u, u1) and same_bits(c, c1)


def test_repeated_device_transports():
    """PEER (fused reduce + finish + all-gather, P2P stores of C) and RED
    (count fan-out) for pass 1; the NCCL transport needs distinct devices
    and is refused cleanly for a repeated one."""
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import GpuError

    d = random_upper(1111, 4)
    u1, c1 = host_call(d)
    for xf in (_lib.EXCHANGE_PEER, _lib.EXCHANGE_RED):
        u, c = host_call(d, devices=[0, 0, 0], xf=xf, xc=_lib.EXCHANGE_PEER)
        assert np.array_equal(u, u1) and same_bits(c, c1), xf
    with pytest.raises(GpuError, match="distinct devices|NCCL"):
        host_call(d, devices=[0, 0], xf=_lib.EXCHANGE_NCCL)


def test_repeated_device_one_sided_and_policies():
    """Tie-heavy integer D (one-sided kernel: each device computes its own
    row band, no pass-2 exchange), InclusiveSplit, and the triplet."""
    d = int_upper(1000, 6)
    for alg, pol in (("pairwise", "strict"), ("pairwise", "split"), ("triplet", "strict")):
        u1, c1 = host_call(d, alg, policy=pol)
        u, c = host_call(d, alg, devices=[0, 0, 0], policy=pol)
        assert np.array_equal(u, u1) and same_bits(c, c1), (alg, pol)
    d = random_upper(1500, 2)
    u1, c1 = host_call(d, "triplet")
    u, c = host_call(d, "triplet", devices=[0, 0, 0, 0])
    assert np.array_equal(u, u1) and same_bits(c, c1)


def test_repeated_device_accurate_and_small():
    from paper_2307_16652_b200 import _lib

    d = random_upper(700, 9)
    u1, c1 = host_call(d, flags=_lib.FLAG_ACCURATE)
    u, c = host_call(d, devices=[0, 0], flags=_lib.FLAG_ACCURATE)
    assert np.array_equal(u, u1) and same_bits(c, c1)
    d = random_upper(130, 9)  # fewer tile rows (2) than devices (3): an empty band
    u1, c1 = host_call(d)
    u, c = host_call(d, devices=[0, 0, 0])
    assert np.array_equal(u, u1) and same_bits(c, c1)


def test_repeated_device_validation_error():
    """A validation error found on the devices comes back as the reference's
    ValidationError with its message, and the next call still works."""
    from paper_2307_16652_b200.api import ValidationError

    d = random_upper(300, 1)
    d[5, 9] = 0.25  # asymmetric: (5, 9) != (9, 5)
    with pytest.raises(ValidationError, match=r"not symmetric at \(5,9\)"):
        host_call(d, devices=[0, 0])
    d = random_upper(300, 1)
    u1, c1 = host_call(d)
    u, c = host_call(d, devices=[0, 0])
    assert np.array_equal(u, u1) and same_bits(c, c1)


def test_cpp_shim_device_list(tmp_path):
    """pald::gpu::parallel_pairwise with a ParallelPlan carrying a device list
    (include/pald_gpu.hpp) == the single-device call, through the C++ shim."""
    import subprocess

    from paper_2307_16652_b200 import _lib

    from test_cpp_shim import build_shim_test

    exe = build_shim_test(tmp_path)
    r = subprocess.run([str(exe), "--devices", "0,0,0"], capture_output=True, text=True, timeout=600,
                       env={"LD_LIBRARY_PATH": str(_lib.LIB_PATH.parent)})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "device list ok" in r.stdout
