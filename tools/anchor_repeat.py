"""Repeatability of the CPU-reference estimator's anchor (bench.py
cpu_reference_sample): estimate / full parallel_pairwise<float> run / estimate
at n = 8192, several times on the box's host cores."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from oracle.oracle import Reference, host_cores  # noqa: E402

ref = Reference()
cores = host_cores()
n = 8192
pts = np.random.default_rng(20230731).random((n, 3))
rc, msg, d64 = ref.points_to_distances(pts)
da = d64.astype(np.float32)
b = ref.default_block_config(4)[0]
ov = ref.pairwise_overhead_f32(n)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    e1, s1 = bench.ref_estimate(ref, da, b, cores, 6.0, ov, rotate=rep)
    _, _, tt = ref.parallel_pairwise(d64, b, cores, use_float=True)
    e2, _ = bench.ref_estimate(ref, da, b, cores, 6.0, ov, rotate=rep + 3, t1=s1["t1"])
    full = float(tt[3])
    print(json.dumps({"rep": rep, "cores": cores, "est_before_s": e1, "full_s": full, "est_after_s": e2,
                      "phase_times_s": [float(x) for x in tt], "overhead_est_s": ov,
                      "rel_error_mean": (0.5 * (e1 + e2) - full) / full, "rel_error_before": (e1 - full) / full}),
          flush=True)
