"""GPU parity: the sm_100a engine (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * U bit-exact (pairwise and triplet, strict-< ties included);
  * pairwise C bit-exact vs the fp32 reference order (blocked_pairwise<float>,
    restated in oracle/pald_oracle.c) -- stronger than the 1e-5 bar;
  * triplet C: max rel_diff (helpers.hpp:30-33 convention) <= 1e-5 vs the
    fp64 oracle, row sums within 1e-5.
"""
import ctypes as C

import numpy as np
import pytest

from helpers import int_upper, max_rel_diff, random_upper

pytestmark = pytest.mark.gpu

TOL = 1e-5


def run_gpu(d: np.ndarray, algorithm: str, force_exact: bool = False):
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for

    lib = _lib.load()
    alg = _lib.PAIRWISE if algorithm == "pairwise" else _lib.TRIPLET
    flags = _lib.FLAG_FORCE_EXACT if force_exact else 0
    opts = _lib.make_opts(algorithm=alg, flags=flags)
    d = np.ascontiguousarray(d, np.float32)
    n = d.shape[0]
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(opts), u.ctypes.data,
                                         c.ctypes.data, None))
    return u, c


SIZES = [2, 3, 5, 16, 33, 65, 127, 128, 129, 200, 257]


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("n", SIZES)
def test_pairwise_bit_exact_random(oracle, n, exact):
    d = random_upper(n, 1000 + n)
    u_ref, c_ref = oracle.pairwise_f32(d)
    u, c = run_gpu(d, "pairwise", exact)
    assert np.array_equal(u, u_ref)
    assert np.array_equal(c.view(np.uint32), c_ref.view(np.uint32))


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("n", [16, 65, 130, 300])
def test_pairwise_bit_exact_ties(oracle, n, exact):
    d = int_upper(n, 77 + n)
    u_ref, c_ref = oracle.pairwise_f32(d)
    u, c = run_gpu(d, "pairwise", exact)
    assert np.array_equal(u, u_ref)
    assert np.array_equal(c.view(np.uint32), c_ref.view(np.uint32))


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("n,kind", [(3, "rand"), (5, "rand"), (33, "rand"), (65, "ties"),
                                    (129, "rand"), (200, "ties"), (257, "rand")])
def test_triplet(oracle, n, kind, exact):
    d = random_upper(n, 2000 + n) if kind == "rand" else int_upper(n, 3000 + n)
    u_ref, c_ref = oracle.triplet_f64(d)
    u, c = run_gpu(d, "triplet", exact)
    assert np.array_equal(u, u_ref)
    assert max_rel_diff(c, c_ref) <= TOL
    assert np.all(np.diagonal(c) == 0.0)
    rs_ref = c_ref.sum(1)
    rs = c.astype(np.float64).sum(1)
    assert np.max(np.abs(rs - rs_ref) / np.maximum(rs_ref, 1.0)) <= TOL


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("n,kind", [(2, "rand"), (3, "t3"), (33, "ties"), (130, "ties"), (200, "rand"), (257, "ties3")])
def test_pairwise_inclusive_split_bit_exact(oracle, n, kind, exact):
    from paper_2307_16652_b200.engine import Engine
    import torch

    if kind == "t3":
        d = np.ones((3, 3), np.float32) - np.eye(3, dtype=np.float32)
    elif kind == "rand":
        d = random_upper(n, 5 + n)
    elif kind == "ties":
        d = int_upper(n, 9 + n)
    else:
        d = int_upper(n, 9 + n, 1, 3)
    u_ref, c_ref = oracle.pairwise_f32(d, policy=1)
    e = Engine(d.shape[0], "pairwise", force_exact=exact, policy="split")
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32))


def _random_case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 420))
    kind = rng.choice(["uniform", "int3", "int16", "points2d", "wide"])
    if kind == "uniform":
        d = random_upper(n, seed)
    elif kind == "int3":
        d = int_upper(n, seed, 1, 3)
    elif kind == "int16":
        d = int_upper(n, seed)
    elif kind == "points2d":
        p = rng.integers(0, 40, size=(n, 2)).astype(np.float64)  # many exact distance ties
        p += rng.random((n, 2)) * 1e-9 * (rng.random() < 0.5)
        diff = p[:, None, :] - p[None, :, :]
        d = np.sqrt((diff ** 2).sum(-1)).astype(np.float32)
        iu = np.triu_indices(n, 1)
        zero = d[iu] == 0
        d[iu[0][zero], iu[1][zero]] = d[iu[1][zero], iu[0][zero]] = 1000.0  # keep D valid
    else:
        d = random_upper(n, seed, 1e-3, 1e3)
    return n, str(kind), d


@pytest.mark.parametrize("seed", list(range(24)))
def test_randomized_sweep(oracle, seed):
    """Random sizes (ragged tiles and chunks) and tie structures through every
    kernel variant: pairwise strict/split and triplet, fast and exact paths."""
    from paper_2307_16652_b200.engine import Engine
    import torch

    n, kind, d = _random_case(seed)
    D = torch.from_numpy(np.ascontiguousarray(d)).cuda()
    exact = bool(seed % 2)
    for policy in ("strict", "split"):
        e = Engine(n, "pairwise", force_exact=exact, policy=policy)
        e.run(D)
        torch.cuda.synchronize()
        u_ref, c_ref = oracle.pairwise_f32(d, policy=0 if policy == "strict" else 1)
        assert np.array_equal(e.U.cpu().numpy(), u_ref), (n, kind, policy)
        assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32)), (n, kind, policy)
    e = Engine(n, "triplet", force_exact=exact)
    e.run(D)
    torch.cuda.synchronize()
    u_ref, c_ref = oracle.triplet_f64(d)
    assert np.array_equal(e.U.cpu().numpy(), u_ref), (n, kind, "triplet")
    assert max_rel_diff(e.C.cpu().numpy(), c_ref) <= TOL, (n, kind, "triplet")


@pytest.mark.parametrize("extreme", ["underflow", "overflow", "both"])
def test_valid_double_inputs_that_degenerate_in_fp32(oracle, extreme):
    """A DistanceMatrix is validated in double (types.hpp:45-65); its fp32
    conversion (to_real<float>, blocked.hpp:91-96) may contain exact 0 or inf
    off the diagonal. The reference float path compares them as is; so must
    we (integer-key path), through the reference-shaped API."""
    import paper_2307_16652_b200 as pg

    n = 97
    rng = np.random.default_rng(5)
    d = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    v = rng.uniform(0.5, 2.0, iu[0].size)
    pick = rng.random(iu[0].size)
    if extreme in ("underflow", "both"):
        v[pick < 0.1] = 1e-50 * (1 + pick[pick < 0.1])  # -> +0.0f
    if extreme in ("overflow", "both"):
        v[pick > 0.9] = 1e300 * (1 + pick[pick > 0.9])  # -> +inf
    d[iu] = v
    d[(iu[1], iu[0])] = v
    dm = pg.DistanceMatrix(n, d)
    d32 = d.astype(np.float32)
    r = pg.blocked_pairwise(dm, 8)
    u_ref, c_ref = oracle.pairwise_f32(d32)
    assert np.array_equal(r.focus.sizes, u_ref)
    # u = 0 pairs (fp32 distance 0) make the reference's masked update add
    # 0*inf = NaN (blocked.hpp:147-148); the NaN rows must coincide
    assert np.array_equal(r.cohesion.values, c_ref.astype(np.float64), equal_nan=True)
    rs = pg.blocked_pairwise(dm, 8, pg.Policy.InclusiveSplit)
    us_ref, cs_ref = oracle.pairwise_f32(d32, policy=1)
    assert np.array_equal(rs.focus.sizes, us_ref)
    assert np.array_equal(rs.cohesion.values, cs_ref.astype(np.float64))
    t = pg.blocked_triplet(dm, 4, 4)
    ut_ref, ct_ref = oracle.triplet_f64(d32)
    assert np.array_equal(t.focus.sizes, ut_ref)
    assert max_rel_diff(t.cohesion.values, ct_ref) <= TOL


def test_device_api_with_leading_dimensions(oracle):
    """pald_gpu_cohesion_f32_device: strided device buffers (ld > n),
    asynchronous on a user stream, U optional."""
    import ctypes as C

    import torch
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for

    lib = _lib.load()
    n = 211
    d = int_upper(n, 12)
    Dbig = torch.zeros((n, n + 13), dtype=torch.float32, device="cuda")
    Dbig[:, :n] = torch.from_numpy(d).cuda()
    U = torch.full((n, n + 5), -7, dtype=torch.int32, device="cuda")
    Cm = torch.full((n, n + 3), 5.0, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for alg in (_lib.PAIRWISE, _lib.TRIPLET):
        opts = _lib.make_opts(algorithm=alg)
        _raise_for(lib.pald_gpu_cohesion_f32_device(Dbig.data_ptr(), n + 13, n, C.byref(opts),
                                                    U.data_ptr(), n + 5, Cm.data_ptr(), n + 3,
                                                    s.cuda_stream))
        s.synchronize()
        if alg == _lib.PAIRWISE:
            u_ref, c_ref = oracle.pairwise_f32(d)
            assert np.array_equal(Cm[:, :n].cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
        else:
            u_ref, c_ref = oracle.triplet_f64(d)
            assert max_rel_diff(Cm[:, :n].cpu().numpy(), c_ref) <= TOL
        assert np.array_equal(U[:, :n].cpu().numpy(), u_ref)
        assert bool((U[:, n:] == -7).all()) and bool((Cm[:, n:] == 5.0).all())  # padding untouched
    # U may be NULL
    opts = _lib.make_opts()
    _raise_for(lib.pald_gpu_cohesion_f32_device(Dbig.data_ptr(), n + 13, n, C.byref(opts), None, 0,
                                                Cm.data_ptr(), n + 3, None))
    torch.cuda.synchronize()
    # a plan can be loaded from host memory, and re-run
    from paper_2307_16652_b200.engine import Engine

    e = Engine(n, "pairwise")
    for _ in range(2):
        e.load_host(np.ascontiguousarray(d))
        e.focus()
        e.cohesion()
    torch.cuda.synchronize()
    u_ref, c_ref = oracle.pairwise_f32(d)
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32))


@pytest.mark.parametrize("n,kind,alg", [(2500, "rand", "pairwise"), (4200, "rand", "pairwise"),
                                        (2500, "fewties", "pairwise"), (2500, "rand", "triplet"),
                                        (3000, "fewties", "triplet"), (2176, "rand", "pairwise"),
                                        (2176, "rand", "triplet"), (8192, "rand", "pairwise")])
def test_host_api_pair_bands_match_one_sided(n, kind, alg):
    """The one-shot host API runs the pair kernel in bands of raster groups
    on two streams with the D2H of finished row bands overlapped, and the
    engine's full-range pass 2 runs it with the last partial round as
    64-wide one-sided tiles (n = 2176: 153 pairs = 148 + 5; n = 8192: 2080 =
    14 x 148 + 8); both must equal the one-sided kernel (engine row ranges)
    bit for bit, at sizes with several raster groups (nb > 16)."""
    import torch

    from paper_2307_16652_b200.engine import Engine

    d = random_upper(n, 11)
    if kind == "fewties":
        d = (np.round(d * 512) / 512).astype(np.float32)
    u, c = run_gpu(d, alg)
    eng = Engine(n, alg)
    eng.load(torch.from_numpy(d).cuda())
    eng.focus()
    h = (n // 2) // 128 * 128
    eng.cohesion(0, h)  # partial row ranges: the one-sided kernel
    eng.cohesion(h, n)
    torch.cuda.synchronize()
    assert eng.info()["cohesion_kernel"].startswith("pald_tile_kernel")
    assert np.array_equal(u, eng.U.cpu().numpy())
    c_bands = eng.C.cpu().numpy()
    assert np.array_equal(c.view(np.uint32), c_bands.view(np.uint32))
    eng.C.zero_()
    eng.cohesion()  # full range: pair kernel (+ 64-wide tail tiles)
    torch.cuda.synchronize()
    if kind == "rand" and alg == "pairwise":  # else the cost model may keep the one-sided kernel
        assert eng.info()["cohesion_kernel"] == "pald_sym_cohesion_kernel"
    if alg == "pairwise":
        assert np.array_equal(eng.C.cpu().numpy().view(np.uint32), c_bands.view(np.uint32))
    else:  # triplet full range: last partial round split along k (sums regrouped)
        assert max_rel_diff(eng.C.cpu().numpy(), c_bands) <= TOL


@pytest.mark.parametrize("n,kind", [(2500, "rand"), (2176, "ties"), (4200, "rand")])
def test_triplet_split_last_round(oracle, n, kind):
    """Triplet pass 2 over the full range splits the pairs of the last partial
    round along k (partial tiles summed in a fixed order): U exact, C within
    1e-5 of the fp64 oracle on sampled rows, and the same bits run to run."""
    import torch

    from paper_2307_16652_b200.engine import Engine

    d = random_upper(n, 5) if kind == "rand" else int_upper(n, 5)
    D = torch.from_numpy(d).cuda()
    eng = Engine(n, "triplet")
    eng.run(D)
    torch.cuda.synchronize()
    c1 = eng.C.cpu().numpy().copy()
    eng.run(D)
    torch.cuda.synchronize()
    assert np.array_equal(eng.C.cpu().numpy().view(np.uint32), c1.view(np.uint32))
    rows = np.unique(np.r_[np.arange(0, n, 97), n - 1])
    ur, cr = oracle.triplet_rows_f64(d, rows)
    assert np.array_equal(eng.U.cpu().numpy()[rows], ur)
    assert max_rel_diff(c1[rows], cr) <= TOL


@pytest.mark.parametrize("mutate", ["asym_low", "asym_high", "neg", "diag", "nan", "zero"])
def test_host_api_banded_validation(mutate):
    """The one-shot host API streams D in bands of 2048 rows and checks each
    band as it arrives (symmetry against the rows above): every invalid
    input is still rejected, wherever the defect sits, and the next call on
    the same cached plan is correct."""
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import ValidationError, _raise_for

    lib = _lib.load()
    n = 4200
    d = random_upper(n, 3)
    i, j = (4100, 7) if mutate != "asym_high" else (7, 4100)
    if mutate.startswith("asym"):
        d[i, j] += 1.0
    elif mutate == "neg":
        d[i, j] = d[j, i] = -1.0
    elif mutate == "diag":
        d[i, i] = 1.0
    elif mutate == "nan":
        d[i, j] = d[j, i] = np.nan
    else:
        d[i, j] = d[j, i] = 0.0
    opts = _lib.make_opts(algorithm=_lib.PAIRWISE)
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    with pytest.raises(ValidationError):
        _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(opts), u.ctypes.data, c.ctypes.data, None))
    good = random_upper(n, 4)
    u2, c2 = run_gpu(good, "pairwise")
    from paper_2307_16652_b200.engine import Engine
    import torch

    e = Engine(n, "pairwise")
    e.run(torch.from_numpy(good).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(u2, e.U.cpu().numpy())
    assert np.array_equal(c2.view(np.uint32), e.C.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("case", ["force_exact", "degenerate"])
def test_host_api_banded_matches_engine_special_layouts(case):
    """The banded host path ranks the raw fp32 bits (sign masked) before the
    range check; with the exact (integer-key) layout for pass 2 (forced, or
    chosen because the fp32 conversion of a valid double input holds 0 and
    inf off the diagonal, validation done in double) it must still equal the
    engine's path (layout keys) bit for bit, NaN rows included."""
    import torch

    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for
    from paper_2307_16652_b200.engine import Engine

    n = 2300
    rng = np.random.default_rng(9)
    d = random_upper(n, 9)
    flags = _lib.FLAG_FORCE_EXACT
    if case == "degenerate":
        iu = np.triu_indices(n, 1)
        pick = rng.random(iu[0].size)
        v = d[iu].copy()
        v[pick < 0.01] = 0.0
        v[pick > 0.99] = np.inf
        d[iu] = v
        d[(iu[1], iu[0])] = v
        flags = _lib.FLAG_SKIP_VALIDATION
    lib = _lib.load()
    opts = _lib.make_opts(algorithm=_lib.PAIRWISE, flags=flags)
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(opts), u.ctypes.data, c.ctypes.data, None))
    e = Engine(n, "pairwise", force_exact=(case == "force_exact"), skip_validation=(case == "degenerate"))
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    assert e.exact_path
    assert np.array_equal(u, e.U.cpu().numpy())
    assert np.array_equal(c, e.C.cpu().numpy(), equal_nan=True)


def test_cached_plan_strict_then_split():
    """The one-shot API caches one plan per device and size: a strict call
    (tie masks, pair kernel) followed by an InclusiveSplit call of the same
    n must run the split semantics (one-sided kernel), equal to a plan made
    for InclusiveSplit."""
    import torch

    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for
    from paper_2307_16652_b200.engine import Engine

    n = 2500
    # a few duplicates per column: the pair kernel stays preferred for strict,
    # and InclusiveSplit differs from strict on those ties
    d = (np.round(random_upper(n, 21) * 2 ** 20) / 2 ** 20).astype(np.float32)
    lib = _lib.load()
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    for policy in (_lib.STRICT, _lib.INCLUSIVE_SPLIT):
        opts = _lib.make_opts(algorithm=_lib.PAIRWISE, policy=policy)
        _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(opts), u.ctypes.data, c.ctypes.data, None))
    e = Engine(n, "pairwise", policy="split")
    D = torch.from_numpy(d).cuda()
    e.run(D)
    torch.cuda.synchronize()
    assert np.array_equal(u, e.U.cpu().numpy())
    assert np.array_equal(c.view(np.uint32), e.C.cpu().numpy().view(np.uint32))
    # the device-pointer API (load through the range check + layout path)
    Ud = torch.empty((n, n), dtype=torch.int32, device="cuda")
    Cd = torch.empty((n, n), dtype=torch.float32, device="cuda")
    for policy in (_lib.STRICT, _lib.INCLUSIVE_SPLIT):
        opts = _lib.make_opts(algorithm=_lib.PAIRWISE, policy=policy)
        _raise_for(lib.pald_gpu_cohesion_f32_device(D.data_ptr(), n, n, C.byref(opts), Ud.data_ptr(), n,
                                                    Cd.data_ptr(), n, None))
        torch.cuda.synchronize()
    assert torch.equal(Ud, e.U)
    assert torch.equal(Cd.view(torch.int32), e.C.view(torch.int32))


def test_cached_plan_split_then_triplet():
    """A plan created for an InclusiveSplit call, reused (same n) for a
    triplet call, must still have the pair kernel's state (tensor maps,
    chunk count) for the triplet's pass 2."""
    import torch

    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for
    from paper_2307_16652_b200.engine import Engine

    n = 2600
    d = random_upper(n, 23)
    lib = _lib.load()
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    for alg, policy in ((_lib.PAIRWISE, _lib.INCLUSIVE_SPLIT), (_lib.TRIPLET, _lib.STRICT)):
        opts = _lib.make_opts(algorithm=alg, policy=policy)
        _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(opts), u.ctypes.data, c.ctypes.data, None))
    e = Engine(n, "triplet")
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(u, e.U.cpu().numpy())
    assert max_rel_diff(c, e.C.cpu().numpy()) <= TOL
