"""Minimal driver for ncu captures of K2 (and friends) at a bench config.

    python tools/profile_k2.py --config 1 --iters 6
Runs one MACE solve warm-up + `iters` timed iterations on the bench plan; prints
the plan info and per-launch K2 timing (CUDA events)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402
from paper_1911_09278_b200.engine import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--sv", type=int, default=8)
ap.add_argument("--schedule", default="sv")
a = ap.parse_args()
c = gen.CONFIGS[a.config]
geom, mats, phantom, y, lam = gen.make_scan(a.config)
N = c["n_agents"]
subs = mb.partition_views(geom.n_views, N)
plan = plan_for(mats, [s.view_indices for s in subs], schedule=a.schedule, sv=a.sv)
prior = mb.PriorParams("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01)
plan.load_data(y, lam)
plan.set_prior(prior)
plan.set_agent_params(-1, c["beta"] / N, 1.0 / c["sigma"] ** 2, False)
plan.stack_init(None, N)
plan.states_from(0)
plan.iterate(3, 0, 0.8, False, 1e-300, N, False)
plan.k2_timing(True)
ms = plan.iterate(a.iters, 3, 0.8, False, 1e-300, N, False)
k2, nl = plan.k2_timing(False)
print("ctx", plan.info())
print("agent0", plan.agent_info(0))
print(f"iterations {a.iters}: {ms:.3f} ms total, K2 {k2 / max(nl, 1):.3f} ms/launch over {nl} launches")
