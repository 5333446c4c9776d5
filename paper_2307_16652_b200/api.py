"""Python mirror of the reference PaLD API, backed by the sm_100a engine.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/pald/*.hpp) so that code and tests written
against the reference read the same here:

  DistanceMatrix      types.hpp:43-75   (validation :45-65)
  FocusSizeMatrix     types.hpp:79-86
  CohesionMatrix      types.hpp:90-98
  PaldResult          types.hpp:106-109
  PhaseTimes          types.hpp:114-119
  Policy              types.hpp:34
  ValidationError / UnsupportedPolicyError / IoError   types.hpp:14-25
  blocked_pairwise    blocked.hpp:368-418
  blocked_triplet     blocked.hpp:424-477
  parallel_pairwise   parallel.hpp:159-222   (ParallelPlan parallel.hpp:31-34)
  parallel_triplet    parallel.hpp:257-320
  fill_diagonal / normalize / local_depths   reference.hpp:213-241

The O(n^3) work always runs on the GPU through the C ABI
(include/pald_gpu.h); the engine computes in fp32 (the reference's
``Real=float`` instantiation), so requesting ``real="float64"`` raises
UnsupportedPolicyError instead of silently changing precision.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class Error(RuntimeError):
    """Base of the reference error hierarchy (types.hpp:14-16)."""


class ValidationError(Error):
    """types.hpp:17-19."""


class UnsupportedPolicyError(Error):
    """types.hpp:20-22."""


class IoError(Error):
    """types.hpp:23-25."""


class GpuError(Error):
    """CUDA or communicator failure inside the engine (status 5/6)."""


class Policy(enum.Enum):
    Strict = 0
    InclusiveSplit = 1


def to_string(p: Policy) -> str:
    return "strict" if p is Policy.Strict else "split"


class UpdateStyle(enum.Enum):
    """blocked.hpp:30-32; both styles give identical bits, so it is accepted
    and ignored exactly as the reference's results ignore it."""

    Masked = 0
    Branchy = 1


@dataclass
class ParallelPlan:
    """parallel.hpp:31-34. ``workers`` is validated (>= 1) like the
    reference; on the GPU it does not change the result (nor does it in
    the reference)."""

    workers: int = 1
    deterministic: bool = False


@dataclass
class PhaseTimes:
    focus_seconds: float = 0.0
    cohesion_seconds: float = 0.0
    overhead_seconds: float = 0.0
    total_seconds: float = 0.0


def _raise_for(code: int) -> None:
    if code == _lib.OK:
        return
    msg = _lib.last_error()
    if code == _lib.ERR_VALIDATION:
        raise ValidationError(msg)
    if code == _lib.ERR_UNSUPPORTED:
        raise UnsupportedPolicyError(msg)
    if code == _lib.ERR_IO:
        raise IoError(msg)
    raise GpuError(f"status {code}: {msg}")


def _cpp_to_string(v: float) -> str:
    """std::to_string(double): printf("%f") (types.hpp:57 formats the value so)."""
    if np.isnan(v):
        return "-nan" if np.signbit(v) else "nan"
    if np.isinf(v):
        return "-inf" if v < 0 else "inf"
    return "%f" % v


class DistanceMatrix:
    """Dense symmetric n x n distance matrix, validated as types.hpp:45-65:
    n >= 2, n*n values, zero diagonal, off-diagonal > 0 (rejects 0 and NaN),
    exact symmetry."""

    def __init__(self, n: int, values):
        n = int(n)
        if n < 2:
            raise ValidationError(f"distance matrix needs n >= 2, got n={n}")
        v = np.asarray(values, dtype=np.float64)
        if v.size != n * n:
            raise ValidationError("distance matrix storage size does not match n*n")
        v = v.reshape(n, n)
        # The reference (types.hpp:50-62) scans row by row: (x, x), then
        # (x, y) for y > x (positivity before symmetry), then row x + 1.
        # Report the first violation in that order: key = x * n + y.
        big = n * n
        bad_diag = np.nonzero(np.diagonal(v) != 0.0)[0]
        k_diag = int(bad_diag[0]) * (n + 1) if bad_diag.size else big
        iu = np.triu_indices(n, 1)
        upper = v[iu]
        notpos = np.nonzero(~(upper > 0.0))[0]
        asym = np.nonzero(upper != v.T[iu])[0]
        keys = iu[0].astype(np.int64) * n + iu[1]
        k_np = int(keys[notpos[0]]) if notpos.size else big
        k_as = int(keys[asym[0]]) if asym.size else big
        first = min(k_diag, k_np, k_as)
        if first < big:
            x, y = divmod(first, n)
            if first == k_diag:
                raise ValidationError(f"distance matrix diagonal entry ({x},{x}) is nonzero")
            if first == k_np:
                raise ValidationError(
                    f"off-diagonal distance ({x},{y}) must be positive, got {_cpp_to_string(v[x, y])} "
                    "(duplicate points are rejected)")
            raise ValidationError(f"distance matrix not symmetric at ({x},{y})")
        self._n = n
        self._v = np.ascontiguousarray(v)
        self._v.setflags(write=False)

    def size(self) -> int:
        return self._n

    def __call__(self, x: int, y: int) -> float:
        return float(self._v[x, y])

    def row(self, x: int) -> np.ndarray:
        return self._v[x]

    def values(self) -> np.ndarray:
        return self._v


@dataclass
class FocusSizeMatrix:
    n: int = 0
    sizes: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.int32))

    def at(self, x: int, y: int) -> int:
        return int(self.sizes[x, y])


@dataclass
class CohesionMatrix:
    n: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float64))
    normalized: bool = False

    def at(self, x: int, z: int) -> float:
        return float(self.values[x, z])


@dataclass
class LocalDepthVector:
    depths: np.ndarray


@dataclass
class PaldResult:
    focus: FocusSizeMatrix
    cohesion: CohesionMatrix


def _check_real(real: str) -> None:
    if real not in ("float32", "float"):
        raise UnsupportedPolicyError(
            f"the GPU engine computes in fp32 (Real=float); real={real!r} is not available")


def _run(d: DistanceMatrix, algorithm: int, policy: Policy, blocks: tuple[int, int, int],
         times: PhaseTimes | None, device: int) -> PaldResult:
    lib = _lib.load()
    opts = _lib.make_opts(algorithm=algorithm, policy=policy.value, device=device, block=blocks[0],
                          block_focus=blocks[1], block_cohesion=blocks[2],
                          flags=_lib.FLAG_SKIP_VALIDATION)
    n = d.size()
    dd = np.ascontiguousarray(d.values().astype(np.float32))  # to_real<float>, blocked.hpp:91-96
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    pt = _lib.PhaseTimes()
    rc = lib.pald_gpu_cohesion_f32(dd.ctypes.data, n, C.byref(opts), u.ctypes.data, c.ctypes.data,
                                   C.byref(pt))
    _raise_for(rc)
    if times is not None:
        times.focus_seconds += pt.focus_seconds
        times.cohesion_seconds += pt.cohesion_seconds
        times.overhead_seconds += pt.overhead_seconds
        times.total_seconds = pt.total_seconds
    # collect_result, blocked.hpp:352-359: fp32 C widened to double
    return PaldResult(FocusSizeMatrix(n, u), CohesionMatrix(n, c.astype(np.float64), False))


def _check_policy_type(policy) -> Policy:
    if not isinstance(policy, Policy):
        raise ValidationError(f"unknown policy {policy!r}")
    return policy


def blocked_pairwise(d: DistanceMatrix, b: int, policy: Policy = Policy.Strict,
                     times: PhaseTimes | None = None, style: UpdateStyle = UpdateStyle.Masked,
                     real: str = "float32", device: int = -1) -> PaldResult:
    """blocked.hpp:368-418 on the GPU."""
    _check_real(real)
    policy = _check_policy_type(policy)
    if b < 1:
        raise ValidationError("pairwise block size must be >= 1")
    return _run(d, _lib.PAIRWISE, policy, (int(b), 128, 128), times, device)


def blocked_triplet(d: DistanceMatrix, b_focus: int, b_cohesion: int,
                    policy: Policy = Policy.Strict, times: PhaseTimes | None = None,
                    style: UpdateStyle = UpdateStyle.Masked, real: str = "float32",
                    device: int = -1) -> PaldResult:
    """blocked.hpp:424-477 on the GPU (C diagonal left 0)."""
    _check_real(real)
    policy = _check_policy_type(policy)
    if policy is not Policy.Strict:
        raise UnsupportedPolicyError("the triplet algorithm supports the strict policy only")
    if b_focus < 1 or b_cohesion < 1:
        raise ValidationError("triplet block sizes must be >= 1")
    return _run(d, _lib.TRIPLET, policy, (128, int(b_focus), int(b_cohesion)), times, device)


def parallel_pairwise(d: DistanceMatrix, b: int, plan: ParallelPlan,
                      policy: Policy = Policy.Strict, times: PhaseTimes | None = None,
                      style: UpdateStyle = UpdateStyle.Masked, real: str = "float32",
                      device: int = -1) -> PaldResult:
    """parallel.hpp:159-222 on the GPU (bit-identical to blocked_pairwise,
    as in the reference, test_parallel.cpp:61-76)."""
    if plan.workers < 1:
        raise ValidationError("worker count must be >= 1")
    if b < 1:
        raise ValidationError("pairwise block size must be >= 1")
    return blocked_pairwise(d, b, policy, times, style, real, device)


def parallel_triplet(d: DistanceMatrix, b_focus: int, b_cohesion: int, plan: ParallelPlan,
                     policy: Policy = Policy.Strict, times: PhaseTimes | None = None,
                     style: UpdateStyle = UpdateStyle.Masked, real: str = "float32",
                     device: int = -1) -> PaldResult:
    """parallel.hpp:257-320 on the GPU."""
    policy = _check_policy_type(policy)
    if policy is not Policy.Strict:
        raise UnsupportedPolicyError("the triplet algorithm supports the strict policy only")
    if plan.workers < 1:
        raise ValidationError("worker count must be >= 1")
    return blocked_triplet(d, b_focus, b_cohesion, policy, times, style, real, device)


def fill_diagonal(u: FocusSizeMatrix, c: CohesionMatrix) -> None:
    """reference.hpp:213-220: c_xx = sum_{y != x} 1/u_xy in double
    (ascending y). Runs on the GPU (pald_gpu_fill_diagonal)."""
    import torch

    lib = _lib.load()
    n = c.n
    du = torch.as_tensor(np.ascontiguousarray(u.sizes, dtype=np.int32)).cuda()
    out = torch.empty(n, dtype=torch.float64, device=du.device)
    stream = torch.cuda.current_stream(du.device).cuda_stream
    _raise_for(lib.pald_gpu_fill_diagonal(du.data_ptr(), n, n, out.data_ptr(), stream))
    diag = out.cpu().numpy()
    c.values[np.arange(n), np.arange(n)] = diag


def _device_values(c: CohesionMatrix):
    import torch

    return torch.from_numpy(np.ascontiguousarray(c.values, np.float64)).cuda()


def normalize(c: CohesionMatrix) -> None:
    """reference.hpp:223-228: c *= 1/(n-1) in double, on the GPU
    (pald_gpu_normalize_f64)."""
    import torch

    if c.normalized:
        raise ValidationError("cohesion matrix is already normalized")
    lib = _lib.load()
    dv = _device_values(c)
    _raise_for(lib.pald_gpu_normalize_f64(dv.data_ptr(), c.n, c.n,
                                          torch.cuda.current_stream(dv.device).cuda_stream))
    c.values = dv.cpu().numpy().reshape(c.n, c.n)
    c.normalized = True


def local_depths(c: CohesionMatrix) -> LocalDepthVector:
    """reference.hpp:231-241: the ascending-z double row sums of a
    normalized C, on the GPU (pald_gpu_row_sums_f64, the reference's order)."""
    import torch

    if not c.normalized:
        raise ValidationError("local depths require a normalized cohesion matrix")
    lib = _lib.load()
    dv = _device_values(c)
    out = torch.empty(c.n, dtype=torch.float64, device=dv.device)
    _raise_for(lib.pald_gpu_row_sums_f64(dv.data_ptr(), c.n, c.n, out.data_ptr(),
                                         torch.cuda.current_stream(dv.device).cuda_stream))
    return LocalDepthVector(out.cpu().numpy())
