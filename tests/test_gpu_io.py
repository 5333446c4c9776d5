"""The reference's binary matrix format read on the GPU, against the
reference's own reader (oracle/_ref: read_distance_binary, ingest.hpp:280)."""
import numpy as np
import pytest
import torch

from helpers import int_upper, random_upper

pytestmark = pytest.mark.gpu


def _sym(n, seed):
    return random_upper(n, seed).astype(np.float64)


CASES = {
    "ok": lambda: _sym(37, 1),
    "ties": lambda: int_upper(40, 2).astype(np.float64),
    "asym_within": lambda: (lambda d: (d.__setitem__((3, 9), d[3, 9] * (1 + 4e-10)), d)[1])(_sym(30, 3)),
    "asym_beyond": lambda: (lambda d: (d.__setitem__((3, 9), d[3, 9] * (1 + 1e-6)), d)[1])(_sym(30, 4)),
    "negative": lambda: (lambda d: (d.__setitem__((5, 2), -1.0), d)[1])(_sym(30, 5)),
    "nonfinite": lambda: (lambda d: (d.__setitem__((7, 1), np.inf), d)[1])(_sym(30, 6)),
    "nan": lambda: (lambda d: (d.__setitem__((2, 8), np.nan), d)[1])(_sym(30, 6)),
    "diag": lambda: (lambda d: (d.__setitem__((4, 4), 0.5), d)[1])(_sym(30, 7)),
    "zero": lambda: (lambda d: (d.__setitem__((6, 11), 0.0), d.__setitem__((11, 6), 0.0), d)[2])(_sym(30, 8)),
    "n1": lambda: np.zeros((1, 1)),
}


@pytest.mark.parametrize("width", [4, 8])
@pytest.mark.parametrize("case", sorted(CASES))
def test_read_distance_binary_matches_reference(reference, tmp_path, case, width):
    from paper_2307_16652_b200 import ValidationError
    from paper_2307_16652_b200.io import read_distance_binary, write_matrix_binary

    d = CASES[case]()
    path = tmp_path / f"{case}_{width}.bin"
    write_matrix_binary(str(path), d, width)
    rc, msg, ref = reference.read_distance_binary(path)
    if rc:
        with pytest.raises(ValidationError) as ei:
            read_distance_binary(str(path))
        assert str(ei.value) == msg
    else:
        got = read_distance_binary(str(path)).cpu().numpy()
        want = ref.astype(np.float32)  # to_real<float>
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_binary_io_errors(tmp_path):
    from paper_2307_16652_b200 import IoError, ValidationError
    from paper_2307_16652_b200.io import read_distance_binary, write_matrix_binary

    with pytest.raises(IoError):
        read_distance_binary(str(tmp_path / "missing.bin"))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValidationError, match="bad magic"):
        read_distance_binary(str(bad))
    p = tmp_path / "trunc.bin"
    write_matrix_binary(str(p), random_upper(20, 1).astype(np.float64), 4)
    p.write_bytes(p.read_bytes()[:-7])
    with pytest.raises(ValidationError, match="truncated payload"):
        read_distance_binary(str(p))
    # corrupt header: n = 2^32 (n * n * width wraps to 0 in 64 bits) and
    # n = 2^20 with a 20-point payload -- refused before anything is allocated
    import struct

    body = p.read_bytes()[14:]
    for n_bad in (1 << 32, 1 << 20):
        h = tmp_path / "hdr.bin"
        h.write_bytes(b"PALD" + struct.pack("<BBQ", 1, 4, n_bad) + body)
        with pytest.raises(ValidationError, match="truncated payload"):
            read_distance_binary(str(h))


def test_binary_to_engine_end_to_end(oracle, tmp_path):
    from paper_2307_16652_b200.engine import Engine
    from paper_2307_16652_b200.io import read_distance_binary, write_matrix_binary

    d = int_upper(300, 4).astype(np.float64)
    p = tmp_path / "d.bin"
    write_matrix_binary(str(p), d, 4)
    D = read_distance_binary(str(p))
    e = Engine(300, "pairwise", skip_validation=True)
    e.run(D)
    torch.cuda.synchronize()
    u_ref, c_ref = oracle.pairwise_f32(d.astype(np.float32))
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
