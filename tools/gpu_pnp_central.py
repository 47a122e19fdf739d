"""Converged MACE-PnP fixed point for config 3 (8 view agents + the 17-layer CNN denoiser, K5),
certified by its equilibrium residuals (mace.py:407-454): the CPU oracle of PnP at 512^2 (torch
CNN on the host, ~1 s per denoise, thousands of iterations) does not finish in a round, so this is
the SURVEY §8c fallback for c3, like tools/gpu_central.py for c2.

Runs PnP MACE on the device (denoiser inside the loop) for --iters iterations from w = 0,
records the Mann relnorm curve and the image H(wbar) at checkpoints, then solves every agent's
proximal map at the final stack to tolerance on the GPU (equilibrium_residuals: r_F = max_i
|F_i(w_i) - x| / |x|, r_u = |H(x + mean(w - x)) - x| / |x|), and the NRMSE of each checkpoint
against the final image (time-to-NRMSE 1e-3 in iterations).

    python tools/gpu_pnp_central.py --iters 4000 --out tests/golden/central_c3.npz
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
from paper_1911_09278_b200.denoisers import CnnDenoiser, DenoiserSpec  # noqa: E402
from paper_1911_09278_b200.engine import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=4000)
ap.add_argument("--every", type=int, default=20)
ap.add_argument("--out", default="")
ap.add_argument("--residuals", type=int, default=1, help="solve the agents' proximal maps at the end")
a = ap.parse_args()
c = gen.CONFIGS[3]
geom, mats, phantom, y, lam = gen.make_scan(3)
N, n = c["n_agents"], geom.n_pixels
prior = mb.PriorParams("qggmrf", beta=c["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
prob = mb.ReconProblem(geom, mats, y, lam, prior)
subs = mb.partition_views(geom.n_views, N)
plan = plan_for(mats, [s.view_indices for s in subs], schedule="sv", sv=8)
den = CnnDenoiser(geom.n_side, seed=0)
sigma_a = np.sqrt(N) * c["sigma"]  # PnP agents: sqrt(N) sigma, beta = 0 (mace.py:263-265)
plan.load_data(y, lam)
plan.set_prior(prior)
plan.set_agent_params(-1, 0.0, 1.0 / sigma_a ** 2, False)
plan.stack_init(None, N)
den.device_apply(plan)
plan.states_from(1)
t = time.time()
snaps, it = {}, 0
while it < a.iters:
    k = min(a.every, a.iters - it)
    plan.iterate(k, it, 0.8, True, 1e-300, N, False, device_denoise=True)
    it += k
    snaps[it] = plan.get_image(1).astype(np.float64)
lg, done = plan.read_log(a.iters)
print(f"{a.iters} PnP iterations in {time.time() - t:.1f} s; done {list(done)}; relnorm first/last "
      f"{lg[0, 0]:.3e} / {lg[-1, 0]:.3e}", flush=True)
x = snaps[a.iters]
nr = {k: float(np.linalg.norm(v - x) / np.linalg.norm(x)) for k, v in snaps.items()}
ks = sorted(nr)
first = next((k for i, k in enumerate(ks) if all(nr[j] <= 1e-3 for j in ks[i:])), None)
q = ks[3 * len(ks) // 4]
print(f"NRMSE vs the final image: <= 1e-3 from iteration {first}; at {q}: {nr[q]:.3e}; "
      f"at {ks[len(ks) // 2]}: {nr[ks[len(ks) // 2]]:.3e}", flush=True)
stack = plan.get_stack().astype(np.float64)
r_F = r_u = float("nan")
if a.residuals:
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=c["sigma"], mode="pnp", max_outer=1, residuals="none",
                        denoiser=DenoiserSpec())  # the spec is unused: the CNN instance is passed below
    t = time.time()
    try:
        res = mb.equilibrium_residuals(prob, cfg, stack, prox_tol=1e-7, denoiser=den)
        r_F, r_u = res.r_F, res.r_u
        print(f"equilibrium residuals (GPU prox solves, {time.time() - t:.1f} s): r_F = {r_F:.3e}, "
              f"r_u = {r_u:.3e}, per agent {[f'{v:.2e}' for v in res.per_agent]}", flush=True)
    except mb.ConvergenceError as err:
        print("equilibrium residuals: a proximal solve did not converge:", err, flush=True)
# drift certificate: change of H(wbar) over the last quarter / half of the run
for frac in (0.5, 0.75, 0.9):
    k = ks[int(frac * (len(ks) - 1))]
    print(f"NRMSE(x_{k}, x_{a.iters}) = {nr[k]:.3e}", flush=True)
if a.out:
    np.savez_compressed(a.out, image=x.astype(np.float32), iterations=a.iters, relnorm=lg[:, 0], r_F=r_F,
                        r_u=r_u, ttr_iterations=-1 if first is None else first, sigma=c["sigma"],
                        how="GPU MACE-PnP with the K5 CNN to convergence, certified by equilibrium residuals "
                            "(tools/gpu_pnp_central.py)")
    print("wrote", a.out)
