"""Converged CPU-oracle MAP image (icd_map_solve restatement) for a bench config.

Writes tests/golden/central_c{config}.npz (float32 image + metadata) — the
fixed-point reference for the GPU parity test at full size.  Heavy: run in
the build container, minutes per config.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

from paper_1911_09278_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--max-passes", type=int, default=3000)
a = ap.parse_args()
c = gen.CONFIGS[a.config]
t = time.time()
geom, mats, phantom, y, lam = gen.make_scan(a.config)  # native tracer: bit-exact (tests/test_native_host.py)
print("scan", time.time() - t, flush=True)
prior = O.Prior("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01)
t = time.time()
hist = []
x, passes = O.icd_map_solve(mats, y, lam, prior, geom.n_side, tol=a.tol, max_passes=a.max_passes,
                            on_pass=lambda k, r, z: (hist.append(r), print(k, r, time.time() - t, flush=True)
                                                     if k % 10 == 0 else None))
cost = O.likelihood_cost(mats, y, lam, x) + O.prior_cost(x, "qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01, 0, geom.n_side)
out = os.path.join(ROOT, "tests", "golden", f"central_c{a.config}.npz")
np.savez_compressed(out, image=x.astype(np.float32), passes=passes, cost=cost, relnorm=np.array(hist),
                    beta=c["beta"], nrmse_phantom=O.nrmse(x, phantom))
print("wrote", out, "passes", passes, "cost", cost, "seconds", time.time() - t)
