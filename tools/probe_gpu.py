"""GPU stability / convergence probe: sweep sigma (and schedule knobs) for a bench config.

    python tools/probe_gpu.py --config 1 --sigmas 2.5e-4,3.5e-4,5e-4 --iters 300
Prints, per sigma, the Mann relnorm trajectory and (if tests/golden/central_c{C}.npz
exists) the NRMSE to the converged CPU-oracle MAP image."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--sigmas", default="3.5e-4")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--schedule", default="sv")
ap.add_argument("--sv", type=int, default=8)
ap.add_argument("--concurrency", default="")
ap.add_argument("--beta", type=float, default=0.0)
ap.add_argument("--out", default="")
a = ap.parse_args()
c = gen.CONFIGS[a.config]
t = time.time()
geom, mats, phantom, y, lam = gen.make_scan(a.config)
print("scan", round(time.time() - t, 1), "s", flush=True)
beta = a.beta or c["beta"]
prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", beta, 2.0, 1.2, 1.0, 0.01))
ref = None
cpath = os.path.join(ROOT, "tests", "golden", f"central_c{a.config}.npz")
if os.path.exists(cpath) and not a.beta:
    ref = np.load(cpath)["image"].astype(np.float64)
results = []
concs = [float(x) for x in a.concurrency.split(",")] if a.concurrency else [None]
for conc in concs:
    if conc is not None:
        os.environ["MACE_SV_CONCURRENCY"] = str(conc)
        import importlib
        import paper_1911_09278_b200.engine as E
        E.DEFAULT_CONCURRENCY = conc
        E.clear_cache()
    for s in [float(x) for x in a.sigmas.split(",")]:
        cfg = mb.MaceConfig(n_subsets=c["n_agents"], rho=0.8, sigma=s, max_outer=a.iters, tol=1e-300,
                            residuals="none", schedule=a.schedule, sv_side=a.sv)
        t = time.time()
        try:
            res = mb.mace_solve(prob, cfg, ref_image=ref)
        except mb.ConvergenceError as err:
            res = err.last_iterate
        dt = time.time() - t
        if res is None:
            print(f"conc={conc} sigma={s}: diverged (non-finite)", flush=True)
            results.append(dict(conc=conc, sigma=s, diverged=True))
            continue
        rel = [r["relnorm"] for r in res.log.rows]
        nr = [r["nrmse"] for r in res.log.rows] if ref is not None else []
        first = next((i + 1 for i in range(len(nr)) if all(v <= 1e-3 for v in nr[i:])), None) if nr else None
        pick = [k for k in (1, 10, 30, 40, 100, 200, 300, 500, 1000, 2000) if k <= len(rel)]
        print(f"conc={conc} sigma={s} iters={len(rel)} wall={dt:.2f}s device_ms={res.device_ms:.1f} "
              f"relnorm@{pick}={[f'{rel[k-1]:.2e}' for k in pick]} "
              + (f"nrmse@{pick}={[f'{nr[k-1]:.2e}' for k in pick]} first<=1e-3 stays: {first}" if nr else ""),
              flush=True)
        results.append(dict(conc=conc, sigma=s, relnorm=rel, nrmse=nr, first_1e3=first, device_ms=res.device_ms))
if a.out:
    json.dump(results, open(a.out, "w"))
