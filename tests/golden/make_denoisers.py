"""The reference's built-in PnP denoisers (denoisers.py:43-106: quadratic-prox as a dense
Cholesky solve and as CG, boxcar at two radii) and its MACE-PnP fixed point with the quadratic
prox at two partitions (mace.py:385-404; its test_mace.py:298-306) -> tests/golden/golden_denoisers.npz.
Run in the build container (imports the reference package from a /tmp copy).

    python tests/golden/make_denoisers.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference, small_problem  # noqa: E402


def main():
    mt = import_reference()
    from macetomo import denoisers as rden
    from macetomo import mace as rmace

    out = {}
    rng = np.random.default_rng(17)
    for n_side, kind, lam, radius in [(8, "quadratic-prox", 2.0, 1), (80, "quadratic-prox", 0.7, 1),
                                      (13, "boxcar", 1.0, 1), (13, "boxcar", 1.0, 3), (40, "boxcar", 1.0, 2)]:
        v = rng.standard_normal(n_side * n_side)
        spec = rden.DenoiserSpec(kind=kind, lam=lam, radius=radius)
        tag = f"{kind}_{n_side}_{radius}"
        out[f"{tag}_in"], out[f"{tag}_out"] = v, rden.make_denoiser(spec, n_side)(v)
        out[f"{tag}_meta"] = np.array([n_side, lam, radius])
    prob = small_problem(mt, 31, 8, 16, 11, "qggmrf", 1.0, 0.5)
    out["pnp_y"], out["pnp_w"] = prob.y, prob.weights
    spec = rden.DenoiserSpec(kind="quadratic-prox", lam=2.0)
    for n in (1, 4):
        cfg = rmace.MaceConfig(n_subsets=n, rho=0.8, sigma=0.1, mode="pnp", denoiser=spec, tol=1e-11,
                               max_outer=8000, residuals="none")
        out[f"pnp_image_n{n}"] = mt.mace_pnp_solve(prob, cfg).image
    path = os.path.join(HERE, "golden_denoisers.npz")
    np.savez_compressed(path, **out)
    d = np.linalg.norm(out["pnp_image_n1"] - out["pnp_image_n4"]) / np.linalg.norm(out["pnp_image_n1"])
    print("PnP N=1 vs N=4 nrmse", d, "wrote", path)


if __name__ == "__main__":
    main()
