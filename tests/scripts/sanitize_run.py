"""Workload for tests/test_gpu_sanitizer.py under compute-sanitizer: the
hot kernels at the smoke sizes -- n = 193 (fp32 pass 1, one-sided pass 2,
pairwise and triplet, tie-heavy) and n = 2304 (rank-coded pass 1, the
tile-pair pass 2 with tie marks and tail tiles, the split triplet pass 2,
accurate mode), plus the multi-device path on a repeated device."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import int_upper, random_upper  # noqa: E402
from paper_2307_16652_b200 import _lib  # noqa: E402
from paper_2307_16652_b200.api import _raise_for  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402

sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [193, 2304]
for n in sizes:
    for kind, d in (("ties", int_upper(n, 5)), ("rand", random_upper(n, 5))):
        D = torch.from_numpy(d).cuda()
        for alg in ("pairwise", "triplet"):
            for acc in (False, True):
                e = Engine(n, alg, accurate=acc)
                e.run(D)
                torch.cuda.synchronize()
                print(n, kind, alg, "accurate" if acc else "default", e.info()["cohesion_kernel"], flush=True)
                del e
    # one call across a repeated device (peer-pull finish, fused pass 2)
    lib = _lib.load()
    d = random_upper(n, 6)
    o = _lib.make_opts(devices=[0, 0])
    u = np.empty((n, n), np.int32)
    c = np.empty((n, n), np.float32)
    _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, None))
    print(n, "multi-device ok", flush=True)
print("sanitize workload done")
