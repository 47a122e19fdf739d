"""Config-3 (MACE-PnP, 512^2, 720 x 725, N = 8, the 17-layer CNN denoiser) oracle run at full
size: 40 iterations of oracle.mace_run -- the restated _run_outer with raster-order float64 ICD
agents (sqrt(N) sigma, beta = 0, mace.py:263-265) and H = oracle/cnn.py's cnn_apply with
BASELINE's weights (He-normal(seed 0) x 0.1, bf16) -- from w = 0.  Writes
tests/golden/pnp_c3_raster40.npz (image = H(mean w) after 40 iterations, float32, plus the
Mann relnorms).  The scan is traced by the oracle (no CUDA library) with gen.make_scan's data
recipe.  TEST INFRASTRUCTURE; ~3 min on 8 cores.

    python tests/golden/make_pnp_c3.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402  (reference_scan: oracle tracer + gen recipe)
import oracle as O  # noqa: E402
from cnn import cnn_apply  # noqa: E402

ITERS = 40


def main():
    workers = max(1, (os.cpu_count() or 2) - 1)
    t = time.time()
    c, ns, mats, y, lam = bench.reference_scan(3, workers)
    gen = bench.load_gen()
    print(f"scan {time.time() - t:.1f} s", flush=True)
    import importlib.util

    spec = importlib.util.spec_from_file_location("_den", os.path.join(ROOT, "paper_1911_09278_b200", "denoisers.py"))
    den = importlib.util.module_from_spec(spec)
    sys.modules["_den"] = den
    spec.loader.exec_module(den)
    w = den.cnn_weights(0)  # CnnDenoiser(n_side, seed=0)'s weights
    H = lambda v: cnn_apply(np.asarray(v, np.float32), w, ns)  # noqa: E731
    prior = O.Prior("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01)
    agents = O.build_agents(mats, y, lam, c["n_agents"], c["sigma"], prior, ns, pnp=True, workers=workers)
    del mats
    t = time.time()
    run = O.mace_run(agents, ITERS, 0.8, denoiser=H, workers=min(workers, c["n_agents"]))
    print(f"{ITERS} PnP iterations {time.time() - t:.1f} s; relnorm {run.relnorms[-1]:.3e}", flush=True)
    assert not run.diverged and len(run.relnorms) == ITERS
    out = os.path.join(HERE, "pnp_c3_raster40.npz")
    np.savez_compressed(out, image=np.asarray(run.image, np.float32), relnorm=np.array(run.relnorms),
                        iters=ITERS, sigma=c["sigma"], how="oracle.mace_run (raster float64 ICD agents, cnn_apply "
                        "denoiser, seed-0 x 0.1 weights), tests/golden/make_pnp_c3.py")
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
