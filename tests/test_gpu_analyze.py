"""SURVEY 8(f) rows 3-4 pinned to the UNMODIFIED reference (oracle/_ref,
oracle/ref_bridge.cpp): the step before the path -- points_to_distances
(ingest.hpp:303-322), duplicate-point rejection included -- and the steps
after it -- normalize / local_depths (reference.hpp:223-241),
universal_threshold / strong_ties / nearest_neighbors (analyze.hpp:34-75).
Every GPU output is compared bit for bit with the reference's."""
import numpy as np
import pytest
import torch

from helpers import int_upper, random_upper

pytestmark = pytest.mark.gpu

SEED = 20230731


def _pts(kind, n):
    from paper_2307_16652_b200 import datagen

    if kind == "gmm16":
        return datagen.points_gmm(n, SEED)
    return datagen.points_uniform(n, {"u2": 2, "u3": 3}[kind], SEED)


@pytest.mark.parametrize("kind", ["u2", "u3", "gmm16"])
def test_points_to_distances_vs_reference(reference, oracle, kind):
    from paper_2307_16652_b200.engine import points_to_distances

    n = 2500
    pts = _pts(kind, n)
    rc, msg, dref = reference.points_to_distances(pts)
    assert rc == 0, msg
    d_gpu = points_to_distances(torch.from_numpy(pts).cuda()).cpu().numpy()
    ref32 = dref.astype(np.float32)  # to_real<float>
    assert np.array_equal(d_gpu.view(np.uint32), ref32.view(np.uint32))
    d_orc, dup = oracle.points_to_distances(pts, fused=True)
    assert dup is None and np.array_equal(d_orc.view(np.uint32), ref32.view(np.uint32))


def test_duplicate_points_rejected_like_reference(reference):
    from paper_2307_16652_b200.api import ValidationError
    from paper_2307_16652_b200.engine import points_to_distances

    pts = _pts("u3", 400)
    pts[17] = pts[250]
    pts[3] = pts[399]
    pts[90] = pts[3]  # (3, 90), (3, 399), (17, 250), (90, 399): first in x < y order is (3, 90)
    rc, msg, _ = reference.points_to_distances(pts)
    assert rc == 2 and "duplicate points 3 and 90" in msg
    with pytest.raises(ValidationError) as ei:
        points_to_distances(torch.from_numpy(pts).cuda())
    assert str(ei.value) == msg


def _engine(d, alg="pairwise"):
    from paper_2307_16652_b200.engine import Engine

    e = Engine(d.shape[0], alg)
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    return e


@pytest.mark.parametrize("alg", ["pairwise", "triplet"])
@pytest.mark.parametrize("data", ["random", "ties"])
def test_epilogue_vs_reference(reference, alg, data):
    """normalize + local_depths, universal_threshold, strong_ties (own and
    explicit threshold), nearest_neighbors: the GPU epilogue on the fp32 C
    in HBM vs the reference on the same C widened to double (triplet: after
    fill_diagonal, as the CLI applies it, pald.cpp:159-160)."""
    n = 700
    d = random_upper(n, 3) if data == "random" else int_upper(n, 3)
    e = _engine(d, alg)
    c = e.C.cpu().numpy().astype(np.float64)
    diag = None
    if alg == "triplet":
        diag = e.fill_diagonal()
        u = e.U.cpu().numpy()
        reference.fill_diagonal(u, c)
        assert np.array_equal(np.diagonal(c), diag.cpu().numpy())
    c_norm, depths = reference.normalize_and_depths(c)
    # local depths (reference.hpp:231-241)
    dg = e.local_depths(diag).cpu().numpy()
    assert np.array_equal(dg.view(np.uint64), depths.view(np.uint64))
    # universal threshold + strong ties (analyze.hpp:34-53)
    thr, xs, ys, sv = reference.strong_ties(c_norm)
    assert thr == reference.universal_threshold(c_norm)
    gthr, gx, gy, gs = e.strong_ties(diag)
    assert np.float64(gthr).view(np.uint64) == np.float64(thr).view(np.uint64)
    assert np.array_equal(gx.cpu().numpy(), xs.astype(np.int32)) and np.array_equal(gy.cpu().numpy(), ys.astype(np.int32))
    assert np.array_equal(gs.cpu().numpy().view(np.uint64), sv.view(np.uint64))
    t2 = float(np.quantile(c_norm[np.triu_indices(n, 1)], 0.9))
    thr2, xs2, ys2, sv2 = reference.strong_ties(c_norm, t2)
    g2 = e.strong_ties(diag, threshold=t2)
    assert g2[0] == thr2 and np.array_equal(g2[1].cpu().numpy(), xs2.astype(np.int32))
    assert np.array_equal(g2[3].cpu().numpy(), sv2)
    # nearest neighbors (analyze.hpp:60-75): ties broken toward smaller z
    for focus, k in ((0, 5), (n - 1, 40), (n // 2, n - 1), (123, 1), (7, 0)):
        rc, msg, zs, sv = reference.nearest_neighbors(c_norm, focus, k)
        assert rc == 0, msg
        gz, gsv = e.nearest_neighbors(focus, k, diag)
        assert np.array_equal(gz.cpu().numpy(), zs.astype(np.int32)), (focus, k)
        assert np.array_equal(gsv.cpu().numpy().view(np.uint64), sv.view(np.uint64))


def test_nearest_neighbor_errors_like_reference(reference):
    from paper_2307_16652_b200.api import ValidationError

    n = 200
    e = _engine(random_upper(n, 1))
    c_norm, _ = reference.normalize_and_depths(e.C.cpu().numpy().astype(np.float64))
    for focus, k in ((n, 3), (0, n), (n + 5, n + 5)):
        rc, msg, _, _ = reference.nearest_neighbors(c_norm, focus, k)
        assert rc == 2
        with pytest.raises(ValidationError) as ei:
            e.nearest_neighbors(focus, k)
        assert str(ei.value) == msg


def test_python_mirror_normalize_and_depths_vs_reference(reference):
    """api.normalize / api.local_depths (GPU kernels on the mirror's double
    CohesionMatrix) == the reference's, bit for bit."""
    from paper_2307_16652_b200 import api

    n = 600
    d = random_upper(n, 8)
    r = api.blocked_pairwise(api.DistanceMatrix(n, d.astype(np.float64)), 64)
    c_ref, depths_ref = reference.normalize_and_depths(r.cohesion.values)
    api.normalize(r.cohesion)
    assert np.array_equal(r.cohesion.values.view(np.uint64), c_ref.view(np.uint64))
    with pytest.raises(api.ValidationError):
        api.normalize(r.cohesion)
    dep = api.local_depths(r.cohesion).depths
    assert np.array_equal(dep.view(np.uint64), depths_ref.view(np.uint64))


@pytest.mark.parametrize("case", ["diag_after_offdiag", "offdiag_before_diag", "asym_then_negative", "nan"])
def test_device_validation_messages_like_reference(reference, case):
    """The raw C ABI validates on the device (stats_kernel) and reports the
    reference's FIRST violation in its scan order with its exact message,
    coordinates and value included (types.hpp:50-62), both for the
    one-shot host call (banded H2D at n > 2048) and the staged plan."""
    import ctypes as C

    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import ValidationError
    from paper_2307_16652_b200.engine import Engine

    for n in (9, 2600):
        d = random_upper(n, 4).astype(np.float64)
        if case == "diag_after_offdiag":
            d[5, 5] = 1.0
            d[2, 7] = d[7, 2] = -1.5
        elif case == "offdiag_before_diag":
            d[4, 4] = 0.5
            d[1, 8] = 0.25
        elif case == "asym_then_negative":
            d[6, 2] = 3.0
            d[3, 8] = d[8, 3] = 0.0
        else:
            d[0, 4] = d[4, 0] = np.nan
        assert reference.validate(d) == 2
        want = reference.lib.ref_last_error().decode()
        d32 = np.ascontiguousarray(d.astype(np.float32))
        lib = _lib.load()
        o = _lib.make_opts()
        c = np.empty((n, n), np.float32)
        rc = lib.pald_gpu_cohesion_f32(d32.ctypes.data, n, C.byref(o), None, c.ctypes.data, None)
        assert rc == _lib.ERR_VALIDATION and _lib.last_error() == want, (n, _lib.last_error(), want)
        e = Engine(n)
        with pytest.raises(ValidationError) as ei:
            e.load(torch.from_numpy(d32).cuda())
        assert str(ei.value) == want
