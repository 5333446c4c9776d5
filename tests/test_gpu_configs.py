"""GPU parity on the five BASELINE.json configurations (seeded synthetic
inputs, paper_2307_16652_b200/datagen.py), through the engine / C ABI.

Full CPU oracles where they finish in seconds (cfg1, and cfg4 triplet on
sampled rows); elsewhere sampled rows of the O(n^2)-per-row restatements
(bit-exact for pairwise, fp64 for triplet) at tile boundaries plus random
rows, and size-independent properties: U symmetric with 2 <= u <= n,
conservation sum(C) = n(n-1)/2 (triplet after fill_diagonal), fast compare
path == integer-key path bit for bit, scale invariance, staged multi-share
focus == single pass.
"""
import numpy as np
import pytest
import torch

from helpers import int_upper, max_rel_diff, random_upper

pytestmark = pytest.mark.gpu

SEED = 20230731


def gpu_d(cfg_index, n=None):
    from paper_2307_16652_b200 import datagen
    from paper_2307_16652_b200.engine import points_to_distances

    cfg = datagen.config(cfg_index)
    if n is not None:
        import dataclasses

        cfg = dataclasses.replace(cfg, n=n)
    pts = datagen.make_points(cfg, SEED)
    if pts is not None:
        return points_to_distances(torch.from_numpy(pts).cuda()), cfg
    return torch.from_numpy(datagen.make_distances(cfg, SEED)).cuda(), cfg


def run(D, alg, force_exact=False):
    from paper_2307_16652_b200.engine import Engine

    e = Engine(D.shape[0], alg, force_exact=force_exact)
    e.run(D)
    torch.cuda.synchronize()
    return e


def sample_rows(n, k=6, seed=0):
    fixed = [0, 1, 127, 128, 129, n // 2, n - 129, n - 128, n - 2, n - 1]
    rng = np.random.default_rng(seed)
    rows = [r for r in fixed if 0 <= r < n] + list(rng.integers(0, n, k))
    return np.unique(np.array(rows, np.int64))


def check_pairwise_rows(oracle, d_host, U, C, rows):
    ur, cr = oracle.pairwise_rows_f32(d_host, rows)
    assert np.array_equal(U[rows], ur)
    assert np.array_equal(C[rows].view(np.uint32), cr.view(np.uint32))


def check_u_props(U):
    n = U.shape[0]
    assert np.array_equal(U, U.T)
    assert np.all(np.diagonal(U) == 0)
    off = U[~np.eye(n, dtype=bool)]
    assert off.min() >= 2 and off.max() <= n


def test_points_kernel_matches_host():
    from paper_2307_16652_b200 import datagen
    from paper_2307_16652_b200.engine import points_to_distances

    for idx in (1, 2, 5):
        cfg = datagen.config(idx)
        pts = datagen.make_points(cfg, SEED)[:700]
        host = datagen.distances_from_points(pts)
        dev = points_to_distances(torch.from_numpy(pts).cuda()).cpu().numpy()
        assert np.array_equal(dev.view(np.uint32), host.view(np.uint32))


def test_cfg1_pairwise_full(oracle):
    D, cfg = gpu_d(1)
    e = run(D, "pairwise")
    d = D.cpu().numpy()
    u_ref, c_ref = oracle.pairwise_f32(d)
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
    n = cfg.n
    assert abs(float(e.C.double().sum()) - n * (n - 1) / 2) / (n * (n - 1) / 2) < 1e-6


def test_cfg4_ties_pairwise_and_triplet(oracle):
    D, cfg = gpu_d(4)
    d = D.cpu().numpy()
    n = cfg.n
    rows = sample_rows(n, 14)
    ep = run(D, "pairwise")
    Up, Cp = ep.U.cpu().numpy(), ep.C.cpu().numpy()
    check_pairwise_rows(oracle, d, Up, Cp, rows)
    check_u_props(Up)
    et = run(D, "triplet")
    Ut, Ct = et.U.cpu().numpy(), et.C.cpu().numpy()
    ur, cr = oracle.triplet_rows_f64(d, rows)
    assert np.array_equal(Ut[rows], ur)
    assert max_rel_diff(Ct[rows], cr) <= 1e-5
    check_u_props(Ut)
    assert (Up != Ut).mean() > 0.5  # the two tie semantics really differ here
    # exact integer-key path agrees bit for bit
    ex = run(D, "triplet", force_exact=True)
    assert np.array_equal(ex.U.cpu().numpy(), Ut)
    assert np.array_equal(ex.C.cpu().numpy().view(np.uint32), Ct.view(np.uint32))


def test_cfg2_triplet(oracle):
    D, cfg = gpu_d(2)
    d = D.cpu().numpy()
    rows = sample_rows(cfg.n, 4)
    e = run(D, "triplet")
    U, Cm = e.U.cpu().numpy(), e.C.cpu().numpy()
    ur, cr = oracle.triplet_rows_f64(d, rows)
    assert np.array_equal(U[rows], ur)
    assert max_rel_diff(Cm[rows], cr) <= 1e-5
    rs, rs_ref = Cm[rows].astype(np.float64).sum(1), cr.sum(1)
    assert np.max(np.abs(rs - rs_ref) / np.maximum(rs_ref, 1.0)) <= 1e-5
    check_u_props(U)
    # conservation after fill_diagonal (reference.hpp:213-220)
    from paper_2307_16652_b200 import _lib

    diag = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
    assert _lib.load().pald_gpu_fill_diagonal(e.U.data_ptr(), e.ld, cfg.n, diag.data_ptr(), None) == 0
    torch.cuda.synchronize()
    total = float(e.C.double().sum()) + float(diag.sum())
    n = cfg.n
    assert abs(total - n * (n - 1) / 2) / (n * (n - 1) / 2) < 1e-6


def test_cfg3_pairwise_rows_and_exact_path(oracle):
    D, cfg = gpu_d(3)
    d = D.cpu().numpy()
    e = run(D, "pairwise")
    U, Cm = e.U.cpu().numpy(), e.C.cpu().numpy()
    check_pairwise_rows(oracle, d, U, Cm, sample_rows(cfg.n, 4))
    check_u_props(U)
    # the BASELINE tolerance against fp64 accumulation (n = 8192)
    from helpers import max_rel_diff

    rows = np.array([0, cfg.n // 2, cfg.n - 1])
    _, c64 = oracle.pairwise_rows_f64(d, rows)
    assert max_rel_diff(Cm[rows], c64) <= 1e-5
    rs = np.abs(Cm[rows].astype(np.float64).sum(1) - c64.sum(1)) / c64.sum(1)
    assert float(rs.max()) <= 1e-5
    del e
    ex = run(D, "pairwise", force_exact=True)
    assert ex.exact_path
    assert np.array_equal(ex.U.cpu().numpy(), U)
    assert np.array_equal(ex.C.cpu().numpy().view(np.uint32), Cm.view(np.uint32))


@pytest.mark.slow
def test_cfg5_pairwise_sampled(oracle):
    D, cfg = gpu_d(5)
    n = cfg.n
    e = run(D, "pairwise")
    rows = np.array([0, 128, n // 2 + 3, n - 1], np.int64)
    d = D.cpu().numpy()
    Ur = e.U[rows.tolist()].cpu().numpy()
    Cr = e.C[rows.tolist()].cpu().numpy()
    ur, cr = oracle.pairwise_rows_f32(d, rows)
    assert np.array_equal(Ur, ur)
    assert np.array_equal(Cr.view(np.uint32), cr.view(np.uint32))
    # against fp64 accumulation: the reference's (and our identical) fp32 C
    # drifts by the rounding of 32768-term sums (see the triplet test below)
    from helpers import max_rel_diff

    _, c64 = oracle.pairwise_rows_f64(d, rows[:2])
    assert max_rel_diff(Cr[:2], c64) <= 3e-5
    rs = np.abs(Cr[:2].astype(np.float64).sum(1) - c64.sum(1)) / c64.sum(1)
    assert float(rs.max()) <= 1e-5
    total = float(e.C.double().sum())
    assert abs(total - n * (n - 1) / 2) / (n * (n - 1) / 2) < 1e-5
    Ut = e.U
    assert bool((Ut == Ut.T).all())
    off = Ut + torch.eye(n, dtype=torch.int32, device="cuda") * 2
    assert int(off.min()) >= 2 and int(Ut.max()) <= n


@pytest.mark.slow
def test_cfg5_points_triplet_sampled(oracle):
    """The triplet algorithm on config 5's n = 32768 D: rank-coded pass 1 at
    the largest rank size (ranks up to 32767), pass 2 with the split last
    round; sampled rows against the fp64 oracle. U exact; C: every entry is
    one fp32 sum of up to 32768 terms, whose rounding alone reaches ~1.4e-5
    relative at this length (the reference's own fp32 pairwise C vs fp64
    grows the same way: 2.0e-6 at n = 1024 ... 7.8e-6 at 8192, SURVEY 8(c)
    probe 3; the 1e-5 bar is stated for the BASELINE triplet configs,
    n <= 4096), so entries are held to 3e-5 and row sums to 1e-5."""
    from helpers import max_rel_diff

    D, cfg = gpu_d(5)
    n = cfg.n
    e = run(D, "triplet")
    assert e.info()["rank_codes"]
    rows = np.array([n - 1], np.int64)  # one O(n^2) oracle row: ~1 min at n = 32768
    d = D.cpu().numpy()
    ur, cr = oracle.triplet_rows_f64(d, rows)
    assert np.array_equal(e.U[rows.tolist()].cpu().numpy(), ur)
    cg = e.C[rows.tolist()].cpu().numpy()
    assert max_rel_diff(cg, cr) <= 3e-5
    rs_g, rs_o = cg.astype(np.float64).sum(1), cr.sum(1)
    assert float(np.max(np.abs(rs_g - rs_o) / rs_o)) <= 1e-5


def test_scale_invariance():
    """test_reference.cpp:183-194: scaling D leaves U and C bit-identical."""
    d = int_upper(300, 5) * np.float32(0.37)
    base = run(torch.from_numpy(d).cuda(), "pairwise")
    U0, C0 = base.U.cpu().numpy(), base.C.cpu().numpy()
    for k in (-60, 7, 40):
        s = run(torch.from_numpy(d * np.float32(2.0 ** k)).cuda(), "pairwise")
        assert np.array_equal(s.U.cpu().numpy(), U0)
        assert np.array_equal(s.C.cpu().numpy().view(np.uint32), C0.view(np.uint32))


def test_permutation_equivariance():
    """test_reference.cpp:196-211: relabelling points permutes C."""
    n = 257
    d = random_upper(n, 11)
    perm = np.random.default_rng(3).permutation(n)
    dp = np.empty_like(d)
    dp[np.ix_(perm, perm)] = d
    a = run(torch.from_numpy(d).cuda(), "pairwise")
    b = run(torch.from_numpy(dp).cuda(), "pairwise")
    Ca, Cb = a.C.cpu().numpy(), b.C.cpu().numpy()
    assert np.array_equal(a.U.cpu().numpy(), b.U.cpu().numpy()[np.ix_(perm, perm)])
    assert max_rel_diff(Ca, Cb[np.ix_(perm, perm)]) < 1e-5


@pytest.mark.parametrize("alg", ["pairwise", "triplet"])
def test_staged_shares_equal_single_pass(alg):
    """Two focus shares on two plans + summed counts + finish == one pass:
    the multi-GPU decomposition, emulated sequentially on one GPU."""
    from paper_2307_16652_b200.engine import Engine

    n = 700
    D = torch.from_numpy(int_upper(n, 9)).cuda()
    ref = run(D, alg)
    parts = 3
    engines = [Engine(n, alg) for _ in range(parts)]
    for i, e in enumerate(engines):
        e.load(D)
        e.focus_counts(i, parts)
    torch.cuda.synchronize()
    total = engines[0].full_W().clone()
    for e in engines[1:]:
        total += e.full_W()
    bands = [(0, 256), (256, 512), (512, n)]
    C = torch.empty((n, n), dtype=torch.float32, device="cuda")
    for e, (r0, r1) in zip(engines, bands):
        e.full_W().copy_(total)
        e.focus_finish()
        e.cohesion(r0, r1)
        torch.cuda.synchronize()
        C[r0:r1] = e.C[r0:r1]
        assert torch.equal(e.U, ref.U)
    assert torch.equal(C.view(torch.int32), ref.C.view(torch.int32))


def test_exact_path_on_wide_range(oracle):
    """Dynamic range beyond the FFMA.SAT compare window -> integer-key path,
    still bit-exact."""
    n = 200
    rng = np.random.default_rng(1)
    d = np.zeros((n, n), np.float32)
    iu = np.triu_indices(n, 1)
    v = (10.0 ** rng.uniform(-30, 30, iu[0].size)).astype(np.float32)
    d[iu] = v
    d[(iu[1], iu[0])] = v
    e = run(torch.from_numpy(d).cuda(), "pairwise")
    assert e.exact_path
    u_ref, c_ref = oracle.pairwise_f32(d)
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
    et = run(torch.from_numpy(d).cuda(), "triplet")
    ut, ct = oracle.triplet_f64(d)
    assert np.array_equal(et.U.cpu().numpy(), ut)
    assert max_rel_diff(et.C.cpu().numpy(), ct) <= 1e-5


def test_validation_errors():
    from paper_2307_16652_b200 import ValidationError
    from paper_2307_16652_b200.engine import Engine

    n = 64
    good = random_upper(n, 1)
    for mutate in ("asym", "neg", "diag", "nan", "zero"):
        d = good.copy()
        if mutate == "asym":
            d[3, 7] += 1.0
        elif mutate == "neg":
            d[3, 7] = d[7, 3] = -1.0
        elif mutate == "diag":
            d[5, 5] = 1.0
        elif mutate == "nan":
            d[3, 7] = d[7, 3] = np.nan
        else:
            d[3, 7] = d[7, 3] = 0.0
        e = Engine(n, "pairwise")
        with pytest.raises(ValidationError):
            e.load(torch.from_numpy(d).cuda())
    # -0.0 on the diagonal is accepted (types.hpp:51)
    d = good.copy()
    d[4, 4] = -0.0
    Engine(n, "pairwise").load(torch.from_numpy(d).cuda())


def test_fill_diagonal_matches_reference_order(oracle):
    from paper_2307_16652_b200 import _lib

    d = int_upper(333, 2)
    e = run(torch.from_numpy(d).cuda(), "triplet")
    out = torch.empty(333, dtype=torch.float64, device="cuda")
    assert _lib.load().pald_gpu_fill_diagonal(e.U.data_ptr(), e.ld, 333, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    u = e.U.cpu().numpy()
    c = np.zeros((333, 333))
    oracle.fill_diagonal(u, c)
    assert np.array_equal(out.cpu().numpy(), np.diagonal(c))


def test_python_api_mirror(oracle):
    """The reference-shaped Python API (DistanceMatrix -> PaldResult)."""
    import paper_2307_16652_b200 as pg

    d32 = random_upper(90, 8)
    dm = pg.DistanceMatrix(90, d32.astype(np.float64))
    r = pg.blocked_pairwise(dm, 16)
    u_ref, c_ref = oracle.pairwise_f32(d32)
    assert np.array_equal(r.focus.sizes, u_ref)
    assert np.array_equal(r.cohesion.values, c_ref.astype(np.float64))
    assert not r.cohesion.normalized
    t = pg.parallel_triplet(dm, 8, 4, pg.ParallelPlan(4, True))
    pg.fill_diagonal(t.focus, t.cohesion)
    assert max_rel_diff(t.cohesion.values, c_ref) < 1e-5  # distinct distances: tri+fill == pairwise
    pg.normalize(r.cohesion)
    assert abs(pg.local_depths(r.cohesion).depths.mean() - 0.5) < 1e-6


@pytest.mark.parametrize("alg", ["pairwise", "triplet"])
def test_epilogue_depths_and_strong_ties(oracle, alg):
    """normalize + local_depths (reference.hpp:223-241) and strong ties
    (analyze.hpp:34-53) on the device, against the reference arithmetic in
    double (the C oracle for depths; a literal restatement for ties)."""
    n = 300
    d = int_upper(n, 21) if alg == "triplet" else random_upper(n, 22)
    e = run(torch.from_numpy(d).cuda(), alg)
    diag = e.fill_diagonal() if alg == "triplet" else None
    depths = e.local_depths(diag).cpu().numpy()
    thr, xs, ys, sv = e.strong_ties(diag)
    c = e.C.cpu().numpy().astype(np.float64)
    if diag is not None:
        np.fill_diagonal(c, diag.cpu().numpy())
    oracle.normalize(c)
    ref_depths = oracle.local_depths(c)
    assert np.array_equal(depths, ref_depths)
    s = 0.0
    for x in range(n):
        s += c[x, x]
    ref_thr = 0.5 * s / n
    assert thr == ref_thr
    edges = [(x, y, min(c[x, y], c[y, x])) for x in range(n) for y in range(x + 1, n)
             if min(c[x, y], c[y, x]) >= ref_thr]
    assert len(edges) == xs.numel() and len(edges) > 0
    got = list(zip(xs.cpu().tolist(), ys.cpu().tolist(), sv.cpu().tolist()))
    assert got == edges
    # explicit threshold override
    thr2, xs2, _, _ = e.strong_ties(diag, threshold=ref_thr * 2)
    assert thr2 == ref_thr * 2 and xs2.numel() == sum(1 for t in edges if t[2] >= ref_thr * 2)


def test_nearest_neighbors_and_normalized(oracle):
    """analyze.hpp:62-75 (stable top-k) and normalize on the device."""
    n = 150
    d = int_upper(n, 31)  # ties in C -> the stable tie-break matters
    e = run(torch.from_numpy(d).cuda(), "pairwise")
    cn = e.normalized_cohesion().cpu().numpy()
    c = e.C.cpu().numpy().astype(np.float64)
    oracle.normalize(c)
    assert np.array_equal(cn, c)
    for focus, k in ((0, 5), (77, 20), (149, 149 - 1)):
        z, s = e.nearest_neighbors(focus, k)
        allz = [(zz, min(c[focus, zz], c[zz, focus])) for zz in range(n) if zz != focus]
        ref = sorted(allz, key=lambda t: -t[1])[:k]  # Python sort is stable
        assert z.cpu().tolist() == [t[0] for t in ref]
        assert s.cpu().tolist() == [t[1] for t in ref]
