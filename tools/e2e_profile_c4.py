"""cProfile of one config-4 mace_solve_batch call (64 slices) after a warm-up call: where the
end-to-end time beyond the device loop goes.  python tools/e2e_profile_c4.py [n_slices]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = gen.CONFIGS[4]
geom, mats, phantoms, ys, lams = gen.make_batch(4, n_slices=S)
prior = mb.PriorParams("qggmrf", beta=cfg["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
probs = [mb.ReconProblem(geom, mats, ys[s], lams[s], prior) for s in range(S)]
mc = mb.MaceConfig(n_subsets=cfg["n_agents"], rho=0.8, sigma=cfg["sigma"], max_outer=30, tol=1e-300,
                   residuals="none")


def solve():
    try:
        return mb.mace_solve_batch(probs, mc)
    except mb.ConvergenceError as e:
        return e.last_iterate


solve()
t0 = time.perf_counter()
res = solve()
print("e2e per batch solve ms", (time.perf_counter() - t0) * 1e3, "device ms", res[0].device_ms)
pr = cProfile.Profile()
pr.enable()
solve()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
