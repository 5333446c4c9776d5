"""ctypes loaders for the CPU oracle and the compiled reference.

TEST INFRASTRUCTURE ONLY. Importable solely from tests/, from
__graft_entry__.smoke() and from bench.py's cpu_baseline / --impl reference
legs -- as the checker or as the timed CPU baseline, never as the product.

* ``Oracle``: oracle/liboracle.so, the C restatement in oracle/pald_oracle.c
  (each function cites the reference file:line it follows).
* ``Reference``: oracle/_ref/libpald_ref_v{3,4}.so, the UNMODIFIED reference
  headers (/root/reference/proj/include) compiled with oracle/ref_bridge.cpp
  by oracle/Makefile. Built in the dev container (where /root/reference
  exists) and carried to the GPU box inside the gpurun snapshot.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_DIR = HERE / "_ref"

_vp, _u64, _i32 = C.c_void_p, C.c_uint64, C.c_int


def build() -> None:
    """Run oracle/Makefile (liboracle.so always; _ref only if the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build()
        lib = C.CDLL(str(ORACLE_SO))
        sigs = {
            "pald_oracle_focus_size": (_i32, [_vp, _u64, _u64, _u64, _i32]),
            "pald_oracle_pairwise_entrywise": (None, [_vp, _u64, _i32, _vp, _vp]),
            "pald_oracle_triplet_entrywise": (_i32, [_vp, _u64, _i32, _vp, _vp]),
            "pald_oracle_fill_diagonal": (None, [_vp, _u64, _vp]),
            "pald_oracle_normalize": (None, [_vp, _u64]),
            "pald_oracle_local_depths": (None, [_vp, _u64, _vp]),
            "pald_oracle_pairwise_f32": (None, [_vp, _u64, _vp, _vp]),
            "pald_oracle_pairwise_policy_f32": (None, [_vp, _u64, _i32, _vp, _vp]),
            "pald_oracle_pairwise_rows_f32": (None, [_vp, _u64, _vp, _u64, _vp, _vp]),
            "pald_oracle_pairwise_f32in_f64": (None, [_vp, _u64, _vp, _vp]),
            "pald_oracle_triplet_f32in_f64": (None, [_vp, _u64, _vp, _vp]),
            "pald_oracle_row_sums_f32": (None, [_vp, _u64, _vp]),
            "pald_oracle_triplet_rows_f64": (None, [_vp, _u64, _vp, _u64, _vp, _vp]),
            "pald_oracle_pairwise_rows_f64": (None, [_vp, _u64, _vp, _u64, _vp, _vp]),
            "pald_oracle_points_to_distances": (C.c_longlong, [_vp, _u64, _u64, _i32, _vp]),
        }
        for k, (r, a) in sigs.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a
        self.lib = lib

    # double-input restatements (reference.hpp)
    def focus_size(self, d: np.ndarray, x: int, y: int, policy: int = 0) -> int:
        d = np.ascontiguousarray(d, np.float64)
        return self.lib.pald_oracle_focus_size(_ptr(d), d.shape[0], x, y, policy)

    def pairwise_entrywise(self, d: np.ndarray, policy: int = 0):
        d = np.ascontiguousarray(d, np.float64)
        n = d.shape[0]
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float64)
        self.lib.pald_oracle_pairwise_entrywise(_ptr(d), n, policy, _ptr(u), _ptr(c))
        return u, c

    def triplet_entrywise(self, d: np.ndarray, validate_ties: bool = False):
        d = np.ascontiguousarray(d, np.float64)
        n = d.shape[0]
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float64)
        rc = self.lib.pald_oracle_triplet_entrywise(_ptr(d), n, int(validate_ties), _ptr(u), _ptr(c))
        if rc:
            raise ValueError("exact distance tie (triplet_entrywise validate_ties)")
        return u, c

    def fill_diagonal(self, u: np.ndarray, c: np.ndarray) -> None:
        assert c.dtype == np.float64
        self.lib.pald_oracle_fill_diagonal(_ptr(np.ascontiguousarray(u, np.int32)), u.shape[0], _ptr(c))

    def normalize(self, c: np.ndarray) -> None:
        self.lib.pald_oracle_normalize(_ptr(c), c.shape[0])

    def local_depths(self, c: np.ndarray) -> np.ndarray:
        out = np.empty(c.shape[0])
        self.lib.pald_oracle_local_depths(_ptr(c), c.shape[0], _ptr(out))
        return out

    # fp32-input restatements
    def pairwise_f32(self, d: np.ndarray, policy: int = 0):
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float32)
        self.lib.pald_oracle_pairwise_policy_f32(_ptr(d), n, policy, _ptr(u), _ptr(c))
        return u, c

    def pairwise_rows_f32(self, d: np.ndarray, rows) -> tuple[np.ndarray, np.ndarray]:
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        rows = np.ascontiguousarray(rows, np.int64)
        u = np.empty((rows.size, n), np.int32)
        c = np.empty((rows.size, n), np.float32)
        self.lib.pald_oracle_pairwise_rows_f32(_ptr(d), n, _ptr(rows), rows.size, _ptr(u), _ptr(c))
        return u, c

    def pairwise_rows_f64(self, d: np.ndarray, rows) -> tuple[np.ndarray, np.ndarray]:
        """Rows of the fp64-accumulated pairwise (Strict) result (tolerance oracle)."""
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        rows = np.ascontiguousarray(rows, np.int64)
        u = np.empty((rows.size, n), np.int32)
        c = np.empty((rows.size, n), np.float64)
        self.lib.pald_oracle_pairwise_rows_f64(_ptr(d), n, _ptr(rows), rows.size, _ptr(u), _ptr(c))
        return u, c

    def triplet_rows_f64(self, d: np.ndarray, rows) -> tuple[np.ndarray, np.ndarray]:
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        rows = np.ascontiguousarray(rows, np.int64)
        u = np.empty((rows.size, n), np.int32)
        c = np.empty((rows.size, n), np.float64)
        self.lib.pald_oracle_triplet_rows_f64(_ptr(d), n, _ptr(rows), rows.size, _ptr(u), _ptr(c))
        return u, c

    def points_to_distances(self, pts: np.ndarray, fused: bool = True):
        """(fp32 D, first duplicate pair or None): ingest.hpp:303-322 as built."""
        pts = np.ascontiguousarray(pts, np.float64)
        n, dim = pts.shape
        out = np.empty((n, n), np.float32)
        k = self.lib.pald_oracle_points_to_distances(_ptr(pts), n, dim, int(fused), _ptr(out))
        return out, (None if k < 0 else divmod(int(k), n))

    def pairwise_f64(self, d: np.ndarray):
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float64)
        self.lib.pald_oracle_pairwise_f32in_f64(_ptr(d), n, _ptr(u), _ptr(c))
        return u, c

    def triplet_f64(self, d: np.ndarray):
        d = np.ascontiguousarray(d, np.float32)
        n = d.shape[0]
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float64)
        self.lib.pald_oracle_triplet_f32in_f64(_ptr(d), n, _ptr(u), _ptr(c))
        return u, c


def _cpu_has_avx512() -> bool:
    try:
        flags = Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    need = ("avx512f", "avx512bw", "avx512dq", "avx512vl")
    return all(f" {f}" in flags for f in need)


class Reference:
    """The unmodified reference library (compiled headers) via ref_bridge.cpp."""

    def __init__(self, path: Path | None = None):
        if path is None:
            v4, v3 = REF_DIR / "libpald_ref_v4.so", REF_DIR / "libpald_ref_v3.so"
            path = v4 if (v4.exists() and _cpu_has_avx512()) else v3
        if not Path(path).exists():
            build()
        if not Path(path).exists():
            raise FileNotFoundError(f"{path}: reference bridge not built (needs /root/reference)")
        self.path = Path(path)
        lib = C.CDLL(str(path))
        d = C.POINTER(C.c_double)
        sigs = {
            "ref_last_error": (C.c_char_p, []),
            "ref_random_distances": (_i32, [_u64, _u64, _vp]),
            "ref_validate": (_i32, [_vp, _u64]),
            "ref_focus_size": (_i32, [_vp, _u64, _u64, _u64, _i32, C.POINTER(C.c_int)]),
            "ref_pairwise_entrywise": (_i32, [_vp, _u64, _i32, _vp, _vp]),
            "ref_triplet_entrywise": (_i32, [_vp, _u64, _i32, _vp, _vp]),
            "ref_oracle_cohesion": (_i32, [_vp, _u64, _i32, _vp]),
            "ref_blocked_pairwise": (_i32, [_vp, _u64, _u64, _i32, _i32, _vp, _vp, _vp]),
            "ref_blocked_triplet": (_i32, [_vp, _u64, _u64, _u64, _i32, _i32, _vp, _vp, _vp]),
            "ref_parallel_pairwise": (_i32, [_vp, _u64, _u64, _i32, _i32, _i32, _vp, _vp, _vp]),
            "ref_parallel_triplet": (_i32, [_vp, _u64, _u64, _u64, _i32, _i32, _i32, _vp, _vp, _vp]),
            "ref_fill_diagonal": (_i32, [_vp, _u64, _vp]),
            "ref_normalize_and_depths": (_i32, [_vp, _u64, _vp]),
            "ref_default_block_config": (_i32, [_u64, _u64, _vp]),
            "ref_read_distance_binary": (_i32, [C.c_char_p, _u64, C.POINTER(C.c_uint64), _vp]),
            "ref_points_to_distances": (_i32, [_vp, _u64, _u64, _vp]),
            "ref_parallel_pairwise_blockpairs_f32": (_i32, [_vp, _u64, _u64, _i32, _vp, _vp, _u64, _vp, _i32, _i32]),
            "ref_pairwise_overhead_f32": (_i32, [_u64, _u64, d]),
            "ref_universal_threshold": (_i32, [_vp, _u64, d]),
            "ref_strong_ties": (_i32, [_vp, _u64, _vp, d, _u64, _vp, _vp, _vp, C.POINTER(C.c_uint64)]),
            "ref_nearest_neighbors": (_i32, [_vp, _u64, _u64, _u64, _vp, _vp]),
        }
        for k, (r, a) in sigs.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a
        self.lib = lib

    def _check(self, rc: int) -> None:
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def random_distances(self, n: int, seed: int) -> np.ndarray:
        out = np.empty((n, n), np.float64)
        self._check(self.lib.ref_random_distances(n, seed, _ptr(out)))
        return out

    def validate(self, d: np.ndarray) -> int:
        d = np.ascontiguousarray(d, np.float64)
        return self.lib.ref_validate(_ptr(d), d.shape[0])

    def _res(self, n):
        return np.empty((n, n), np.int32), np.empty((n, n), np.float64), np.zeros(4)

    def pairwise_entrywise(self, d, policy=0):
        d = np.ascontiguousarray(d, np.float64)
        u, c, _ = self._res(d.shape[0])
        self._check(self.lib.ref_pairwise_entrywise(_ptr(d), d.shape[0], policy, _ptr(u), _ptr(c)))
        return u, c

    def triplet_entrywise(self, d, validate_ties=False):
        d = np.ascontiguousarray(d, np.float64)
        u, c, _ = self._res(d.shape[0])
        self._check(self.lib.ref_triplet_entrywise(_ptr(d), d.shape[0], int(validate_ties), _ptr(u), _ptr(c)))
        return u, c

    def oracle_cohesion(self, d, policy=0):
        d = np.ascontiguousarray(d, np.float64)
        c = np.empty_like(d)
        self._check(self.lib.ref_oracle_cohesion(_ptr(d), d.shape[0], policy, _ptr(c)))
        return c

    def blocked_pairwise(self, d, b, policy=0, use_float=True):
        d = np.ascontiguousarray(d, np.float64)
        u, c, t = self._res(d.shape[0])
        self._check(self.lib.ref_blocked_pairwise(_ptr(d), d.shape[0], b, policy, int(use_float),
                                                  _ptr(u), _ptr(c), _ptr(t)))
        return u, c, t

    def blocked_triplet(self, d, bf, bc, use_float=True):
        d = np.ascontiguousarray(d, np.float64)
        u, c, t = self._res(d.shape[0])
        self._check(self.lib.ref_blocked_triplet(_ptr(d), d.shape[0], bf, bc, 0, int(use_float),
                                                 _ptr(u), _ptr(c), _ptr(t)))
        return u, c, t

    def parallel_pairwise(self, d, b, workers, use_float=True):
        d = np.ascontiguousarray(d, np.float64)
        u, c, t = self._res(d.shape[0])
        self._check(self.lib.ref_parallel_pairwise(_ptr(d), d.shape[0], b, workers, 0, int(use_float),
                                                   _ptr(u), _ptr(c), _ptr(t)))
        return u, c, t

    def parallel_triplet(self, d, bf, bc, workers, use_float=True):
        d = np.ascontiguousarray(d, np.float64)
        u, c, t = self._res(d.shape[0])
        self._check(self.lib.ref_parallel_triplet(_ptr(d), d.shape[0], bf, bc, workers, 0,
                                                  int(use_float), _ptr(u), _ptr(c), _ptr(t)))
        return u, c, t

    def fill_diagonal(self, u, c):
        self._check(self.lib.ref_fill_diagonal(_ptr(np.ascontiguousarray(u, np.int32)), u.shape[0], _ptr(c)))

    def normalize_and_depths(self, c: np.ndarray):
        """reference.hpp:223-241 on a copy of c: (normalized C, local depths)."""
        c = np.array(c, np.float64, order="C", copy=True)
        depths = np.empty(c.shape[0])
        self._check(self.lib.ref_normalize_and_depths(_ptr(c), c.shape[0], _ptr(depths)))
        return c, depths

    def read_distance_binary(self, path, cap=4096):
        """(status, message, D) of the reference's read_distance_binary."""
        n = C.c_uint64(0)
        out = np.empty(cap * cap, np.float64)
        rc = self.lib.ref_read_distance_binary(str(path).encode(), cap, C.byref(n), _ptr(out))
        if rc:
            return rc, self.lib.ref_last_error().decode(), None
        k = int(n.value)
        return 0, "", out[: k * k].reshape(k, k).copy()

    def default_block_config(self, element_bytes=4, cache_bytes=0):
        out = np.zeros(3, np.uint64)
        self._check(self.lib.ref_default_block_config(element_bytes, cache_bytes, _ptr(out)))
        return tuple(int(v) for v in out)

    def parallel_pairwise_blockpairs_f32(self, d32: np.ndarray, b: int, workers: int, pairs) -> np.ndarray:
        """Seconds of each listed block pair (xb, yb) of the parallel_pairwise<float>
        driver loop (ref_bridge.cpp ref_parallel_pairwise_blockpairs_f32)."""
        d32 = np.ascontiguousarray(d32, np.float32)
        pairs = np.asarray(pairs, np.uint32).reshape(-1, 2)
        xb, yb = np.ascontiguousarray(pairs[:, 0]), np.ascontiguousarray(pairs[:, 1])
        out = np.zeros(len(pairs))
        self._check(self.lib.ref_parallel_pairwise_blockpairs_f32(_ptr(d32), d32.shape[0], b, workers, _ptr(xb),
                                                                 _ptr(yb), len(pairs), _ptr(out), 0, 0))
        return out

    def pairwise_overhead_f32(self, n: int, seed: int = 1) -> float:
        """Seconds of the O(n^2) part of a parallel_pairwise<float> call at size n."""
        out = C.c_double(0.0)
        self._check(self.lib.ref_pairwise_overhead_f32(n, seed, C.byref(out)))
        return out.value

    def points_to_distances(self, pts: np.ndarray):
        """(status, message, D double) of ingest.hpp:303-322."""
        pts = np.ascontiguousarray(pts, np.float64)
        n, dim = pts.shape
        out = np.empty((n, n), np.float64)
        rc = self.lib.ref_points_to_distances(_ptr(pts), n, dim, _ptr(out))
        if rc:
            return rc, self.lib.ref_last_error().decode(), None
        return 0, "", out

    def universal_threshold(self, c_norm: np.ndarray) -> float:
        c_norm = np.ascontiguousarray(c_norm, np.float64)
        out = C.c_double(0.0)
        self._check(self.lib.ref_universal_threshold(_ptr(c_norm), c_norm.shape[0], C.byref(out)))
        return out.value

    def strong_ties(self, c_norm: np.ndarray, threshold: float | None = None):
        """(threshold, xs, ys, strength) of analyze.hpp:42-53."""
        c_norm = np.ascontiguousarray(c_norm, np.float64)
        n = c_norm.shape[0]
        thr_in = np.array([threshold if threshold is not None else 0.0])
        thr, cnt = C.c_double(0.0), C.c_uint64(0)
        tp = _ptr(thr_in) if threshold is not None else None
        self._check(self.lib.ref_strong_ties(_ptr(c_norm), n, tp, C.byref(thr), 0, None, None, None,
                                             C.byref(cnt)))
        m = int(cnt.value)
        xs, ys, sv = np.empty(m, np.uint64), np.empty(m, np.uint64), np.empty(m, np.float64)
        self._check(self.lib.ref_strong_ties(_ptr(c_norm), n, tp, C.byref(thr), m, _ptr(xs), _ptr(ys),
                                             _ptr(sv), C.byref(cnt)))
        return thr.value, xs, ys, sv

    def nearest_neighbors(self, c_norm: np.ndarray, focus: int, k: int):
        """(status, message, zs, strength) of analyze.hpp:60-75."""
        c_norm = np.ascontiguousarray(c_norm, np.float64)
        zs, sv = np.empty(max(k, 1), np.uint64), np.empty(max(k, 1), np.float64)
        rc = self.lib.ref_nearest_neighbors(_ptr(c_norm), c_norm.shape[0], focus, k, _ptr(zs), _ptr(sv))
        if rc:
            return rc, self.lib.ref_last_error().decode(), None, None
        return 0, "", zs[:k], sv[:k]


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
