"""Centralized ICD on the parallel super-voxel pass (multi-warp tiles): stability and speed against
the number of tiles in flight and a proximal anchor (each pass targets v = z at the pass start with
weight kappa * mean(theta2); kappa = 0 is plain icd_map_solve).

    python tools/probe_central.py --config 0 --blocks 1,4,16,0 --kappa 0,2,8 --passes 400
Prints passes to NRMSE <= 1e-3 against the CPU-oracle MAP (tests/golden/central_c<config>.npz)."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402
from paper_1911_09278_b200.engine import AgentPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=0)
ap.add_argument("--blocks", default="1,4,16,0")
ap.add_argument("--kappa", default="0,2,8")
ap.add_argument("--passes", type=int, default=400)
ap.add_argument("--schedule", default="sv")
a = ap.parse_args()
c = gen.CONFIGS[a.config]
geom, mats, phantom, y, lam = gen.make_scan(a.config)
ref = np.load(os.path.join(ROOT, "tests", "golden", f"central_c{a.config}.npz"))["image"]
prior = mb.PriorParams("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01)
plan = AgentPlan(mats, [tuple(range(geom.n_views))], schedule=a.schedule)
plan.load_data(y, lam)
plan.set_prior(prior)
th = plan.get_theta2(0).astype(np.float64)
print("info", plan.info(), "mean theta2 %.3e" % th.mean(), flush=True)
for blocks in [int(x) for x in a.blocks.split(",")]:
    for kappa in [float(x) for x in a.kappa.split(",")]:
        ng = -(-geom.n_views // 32)
        chunks = -(-ng // 3) if ng > 4 else 1
        plan.set_schedule(1.0 / 16.0, blocks * chunks)
        plan.set_agent_params(0, prior.beta, kappa * th.mean(), False)
        z = np.zeros(geom.n_pixels)
        plan.set_state(0, z)
        hit, t0, nr = None, time.perf_counter(), np.inf
        for k in range(a.passes):
            dsq = plan.run_pass(0, z)[0]
            if (k + 1) % 50 == 0:
                plan.refresh(0)
            z = plan.get_state(0).astype(np.float64)
            nr = float(np.linalg.norm(z - ref) / np.linalg.norm(ref))
            if not np.isfinite(nr) or nr > 1e3:
                break
            if hit is None and nr <= 1e-3:
                hit = k + 1
        dt = time.perf_counter() - t0
        print(f"config {a.config} blocks {blocks:3d} kappa {kappa:4.1f}: NRMSE {nr:.2e} after {k + 1} passes, "
              f"<=1e-3 at {hit}, {dt / (k + 1) * 1e3:.2f} ms/pass (host loop), {plan.info()['sv_grid']} warps",
              flush=True)
