"""GPU-converged MAP image for a config the CPU oracle cannot converge in a round (config 2),
certified by the MAP-cost gradient (SURVEY §8c fallback: "fixed point verified via cost and
gradient norm").

Runs conventional MACE (SV schedule) for --iters iterations, then reports the stationarity ratio
|grad f(x)| / |grad f(0)| (fp64 accumulation, mace_gradient).  With --calibrate 1 it does the
same at config 1 and also evaluates the ratio at the CPU oracle's float64 MAP
(tests/golden/central_c1.npz), so the c2 ratio can be read against a known-good one.

    python tools/gpu_central.py --config 2 --iters 6000 --out tests/golden/central_c2.npz
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
ap.add_argument("--iters", type=int, default=6000)
ap.add_argument("--out", default="")
a = ap.parse_args()
c = gen.CONFIGS[a.config]
t = time.time()
geom, mats, phantom, y, lam = gen.make_scan(a.config)
print("scan", round(time.time() - t, 1), flush=True)
N, n = c["n_agents"], geom.n_pixels
prior = mb.PriorParams("qggmrf", beta=c["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
prob = mb.ReconProblem(geom, mats, y, lam, prior)
subs = mb.partition_views(geom.n_views, N)
plan = plan_for(mats, [s.view_indices for s in subs], schedule="sv", sv=8)
plan.load_data(y, lam)
plan.set_prior(prior)
plan.set_agent_params(-1, prior.beta / N, 1.0 / c["sigma"] ** 2, False)
plan.stack_init(None, N)
plan.states_from(0)
t = time.time()
checkpoints = {}
done_iters = 0
for stop in sorted({a.iters // 4, a.iters // 2, 3 * a.iters // 4, a.iters}):
    plan.iterate(stop - done_iters, done_iters, 0.8, False, 1e-300, N, False)
    done_iters = stop
    checkpoints[stop] = plan.get_image(0).astype(np.float32)
lg, done = plan.read_log(a.iters)
print("iterations", a.iters, "device+host s", round(time.time() - t, 1), "done", list(done),
      "final relnorm", lg[-1, 0], flush=True)
_, g0 = mb.map_gradient(prob, np.zeros(n, np.float32))
report = {}
for k, x in checkpoints.items():
    _, gk = mb.map_gradient(prob, x)
    report[k] = gk[0] / g0[0]
    print(f"iter {k}: |grad| / |grad(0)| = {gk[0] / g0[0]:.3e} (data {gk[1]:.3e}, prior {gk[2]:.3e})", flush=True)
x = checkpoints[a.iters]
ks = sorted(checkpoints)
drift = float(np.linalg.norm(x - checkpoints[ks[-2]]) / np.linalg.norm(x))
print(f"relative change over the last {a.iters - ks[-2]} iterations: {drift:.3e}")
if a.config == 1:
    ref = np.load(os.path.join(ROOT, "tests", "golden", "central_c1.npz"))["image"]
    _, gr = mb.map_gradient(prob, ref.astype(np.float32))
    print(f"CPU oracle MAP: |grad| / |grad(0)| = {gr[0] / g0[0]:.3e}; nrmse(GPU, CPU) = "
          f"{np.linalg.norm(x - ref) / np.linalg.norm(ref):.3e}")
if a.out:
    np.savez_compressed(a.out, image=x, iterations=a.iters, grad_ratio=report[a.iters], relnorm=lg[:, 0],
                        drift_last_quarter=drift, beta=c["beta"], sigma=c["sigma"],
                        how="GPU MACE (SV schedule) to convergence, certified by |grad f| (tools/gpu_central.py)")
    print("wrote", a.out)
