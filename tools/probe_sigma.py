"""Stability / convergence-speed probe of the proximal sigma on the GPU (SV schedule).

For each sigma and agent-group size (mace_set_agent_groups: 0 = every local agent at once,
g = the per-agent staleness of a rank that owns g agents), runs a fresh MACE solve and
reports the first iteration after which NRMSE against the converged reference image
(tests/golden/central_c{config}.npz) stays <= 1e-3, the final NRMSE, and divergence.

    python tools/probe_sigma.py --config 2 --sigmas 3.5e-4,7e-4,1e-3 --groups 0,2 --iters 8000
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402
from paper_1911_09278_b200.engine import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--sigmas", default="3.5e-4,7e-4,1e-3")
ap.add_argument("--groups", default="0,2")
ap.add_argument("--iters", type=int, default=8000)
ap.add_argument("--ref", default="")
ap.add_argument("--save", default="", help="save the final image of each run here (npz)")
ap.add_argument("--schedule", default="sv", choices=["sv", "sv-det"])
a = ap.parse_args()
c = gen.CONFIGS[a.config]
t = time.time()
geom, mats, phantom, y, lam = gen.make_scan(a.config)
N, n = c["n_agents"], geom.n_pixels
prior = mb.PriorParams("qggmrf", beta=c["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
plan = plan_for(mats, [s.view_indices for s in mb.partition_views(geom.n_views, N)], schedule=a.schedule, sv=8)
plan.load_data(y, lam)
plan.set_prior(prior)
ref = np.load(a.ref or os.path.join(ROOT, "tests", "golden", f"central_c{a.config}.npz"))["image"].astype(np.float32)
print(f"setup {time.time() - t:.1f} s; ref {a.ref or 'central_c%d' % a.config}", flush=True)
saved = {}
for g in [int(x) for x in a.groups.split(",")]:
    if a.schedule == "sv":
        plan.set_agent_groups(g)
    for sg in [float(x) for x in a.sigmas.split(",")]:
        plan.set_agent_params(-1, prior.beta / N, 1.0 / sg ** 2, False)
        plan.set_ref(ref)
        plan.stack_init(None, N)
        plan.states_from(0)
        ms = plan.iterate(a.iters, 0, 0.8, False, 1e-300, N, True)
        lg, done = plan.read_log(a.iters)
        nr = lg[:, 3]
        ran = len(nr) if done[0] == 0 else done[1]
        nr = nr[:ran]
        ok = nr <= 1e-3
        first = next((i + 1 for i in range(len(nr)) if ok[i:].all()), None)
        pts = {k: float(nr[k - 1]) for k in (500, 1000, 2000, 4000, 8000, 16000) if k <= len(nr)}
        print(f"group {g:2d} sigma {sg:.2e}: done {list(done)} first<=1e-3 {first} final nrmse "
              f"{nr[-1] if len(nr) else float('nan'):.3e} min {np.nanmin(nr) if len(nr) else float('nan'):.3e} "
              f"ms/iter {ms / max(ran, 1):.3f}  {pts}", flush=True)
        if a.save:
            saved[f"g{g}_s{sg:.2e}"] = plan.get_image(0).copy()
        plan.set_ref(None)
if a.save:
    np.savez_compressed(a.save, **saved)
