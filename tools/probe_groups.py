"""K2 launch time against the agent-group size of the super-voxel queue (mace_set_agent_groups).

    python tools/probe_groups.py --config 1 --groups 0,1,2,4,8
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402
from paper_1911_09278_b200.engine import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--groups", default="0,1,2,4,8")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sv", type=int, default=8)
a = ap.parse_args()
c = gen.CONFIGS[a.config]
geom, mats, phantom, y, lam = gen.make_scan(a.config)
N = c["n_agents"]
prior = mb.PriorParams("qggmrf", beta=c["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
plan = plan_for(mats, [s.view_indices for s in mb.partition_views(geom.n_views, N)], schedule="sv", sv=a.sv)
plan.load_data(y, lam)
plan.set_prior(prior)
plan.set_agent_params(-1, prior.beta / N, 1.0 / c["sigma"] ** 2, False)
for rep in range(a.reps):
    for g in [int(x) for x in a.groups.split(",")]:
        plan.set_agent_groups(g)
        plan.stack_init(None, N)
        plan.states_from(0)
        plan.iterate(5, 0, 0.8, False, 1e-300, N, False)
        plan.k2_timing(True)
        ms = plan.iterate(a.iters, 0, 0.8, False, 1e-300, N, False)
        k2, nl = plan.k2_timing(False)
        print(f"config {a.config} sv {a.sv} rep {rep} group {g:2d}: K2 {k2 / nl:.4f} ms/launch, loop {ms / a.iters:.4f} ms/iter",
              flush=True)
