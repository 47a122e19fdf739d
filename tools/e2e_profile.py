import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen
import cProfile, pstats
C = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = gen.CONFIGS[C]
geom, mats, ph, y, lam = gen.make_scan(C)
prior = mb.PriorParams("qggmrf", beta=cfg["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
prob = mb.ReconProblem(geom, mats, y, lam, prior)
mc = mb.MaceConfig(n_subsets=cfg["n_agents"], rho=0.8, sigma=cfg["sigma"], max_outer=cfg["iters"], tol=1e-300,
                   residuals="none")
def solve():
    try:
        return mb.mace_solve(prob, mc)
    except mb.ConvergenceError as e:
        return e.last_iterate
for _ in range(2): solve()
t = time.perf_counter()
for _ in range(5): r = solve()
print("e2e per solve ms", (time.perf_counter() - t) / 5 * 1e3, "device ms", r.device_ms)
pr = cProfile.Profile(); pr.enable(); solve(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
