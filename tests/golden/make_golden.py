"""Generate golden vectors from the UNMODIFIED reference (compiled headers,
oracle/_ref via oracle/ref_bridge.cpp). Run in the dev container, where
/root/reference exists:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz. Contents (per case "<name>"):
  <name>.D          float64 n x n input (reference random_distances or fixtures)
  <name>.pw_U/C     pairwise_entrywise(d, Strict)          reference.hpp:104-147
  <name>.pwf_C      blocked_pairwise<float>(d, b=5) C       blocked.hpp:368-418
  <name>.tr_U/C     triplet_entrywise(d)                    reference.hpp:154-208
  <name>.trf_C      blocked_triplet<float>(d, 8, 4) C       blocked.hpp:424-477
  <name>.split_U/C  pairwise_entrywise(d, InclusiveSplit)
  <name>.splitf_C   blocked_pairwise<float>(d, b=5, InclusiveSplit) C
  <name>.fill_C     triplet C after fill_diagonal           reference.hpp:213-220
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference  # noqa: E402


def dmat(n, upper):
    d = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    d[iu] = upper
    d[(iu[1], iu[0])] = upper
    return d


def main():
    ref = Reference()
    cases = {
        "d2": dmat(2, [5.0]),
        "d3": dmat(3, [1.0, 2.0, 3.0]),
        "t3": dmat(3, [1.0, 1.0, 1.0]),
    }
    for n in (5, 16, 33, 65):
        cases[f"rd{n}"] = ref.random_distances(n, 1000 + n)   # test_blocked.cpp:40 seeds
    rng = np.random.default_rng(4242)
    for n in (17, 48):
        iu = np.triu_indices(n, 1)
        cases[f"ties{n}"] = dmat(n, rng.integers(1, 17, iu[0].size).astype(np.float64))
    out = {}
    for name, d in cases.items():
        out[f"{name}.D"] = d
        u, c = ref.pairwise_entrywise(d, 0)
        out[f"{name}.pw_U"], out[f"{name}.pw_C"] = u, c
        _, cf, _ = ref.blocked_pairwise(d, 5, 0, use_float=True)
        out[f"{name}.pwf_C"] = cf
        ut, ct = ref.triplet_entrywise(d)
        out[f"{name}.tr_U"], out[f"{name}.tr_C"] = ut, ct
        _, ctf, _ = ref.blocked_triplet(d, 8, 4, use_float=True)
        out[f"{name}.trf_C"] = ctf
        us, cs = ref.pairwise_entrywise(d, 1)
        out[f"{name}.split_U"], out[f"{name}.split_C"] = us, cs
        _, csf, _ = ref.blocked_pairwise(d, 5, 1, use_float=True)
        out[f"{name}.splitf_C"] = csf
        cfill = ct.copy()
        ref.fill_diagonal(ut, cfill)
        out[f"{name}.fill_C"] = cfill
    path = Path(__file__).resolve().parent / "golden.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes, {len(cases)} cases)")


if __name__ == "__main__":
    main()
