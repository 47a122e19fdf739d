"""Reference equilibrium residuals (mace.py:407-454) and the reference's default
residuals="final" path (mace.py:353-357) on small problems -> tests/golden/golden_residuals.npz.
Run in the build container (imports the reference package from a /tmp copy).

    python tests/golden/make_residuals.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ellipse_problem, import_reference, small_problem  # noqa: E402


def main():
    mt = import_reference()
    from macetomo import icd as ricd
    from macetomo import mace as rmace

    out = {}

    def fixed(fn, prob, cfg, **kw):
        try:
            return fn(prob, cfg, **kw)
        except ricd.ConvergenceError as err:
            return err.last_iterate

    # (a) conventional, mid-run stack (12 iterations): r_F well away from 0
    prob = small_problem(mt, 31, 8, 16, 11, "qggmrf", 1.0, 0.5)
    out["mq_y"], out["mq_w"] = prob.y, prob.weights
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=12, tol=1e-300, residuals="none")
    w12 = fixed(mt.mace_solve, prob, cfg).stack
    rep = mt.mace.equilibrium_residuals(prob, cfg, w12)
    out["a_stack"], out["a_rF"], out["a_ru"], out["a_per_agent"] = w12, rep.r_F, rep.r_u, np.array(rep.per_agent)
    # (b) the reference default: residuals="final" after convergence
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=8000, tol=1e-9)
    res = mt.mace_solve(prob, cfg)
    out["b_stack"], out["b_image"] = res.stack, res.image
    out["b_rF"], out["b_ru"], out["b_iters"] = res.residuals.r_F, res.residuals.r_u, res.iterations
    out["b_per_agent"] = np.array(res.residuals.per_agent)
    # (c) counts-weighted ellipse problem (config-0 recipe in miniature), mid-run stack
    eprob, _ = ellipse_problem(mt, 32, 45, 47, seed=3, beta=20.0)
    out["ell_y"], out["ell_w"] = eprob.y, eprob.weights
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=3e-4, max_outer=30, tol=1e-300, residuals="none")
    w30 = fixed(mt.mace_solve, eprob, cfg).stack
    rep = mt.mace.equilibrium_residuals(eprob, cfg, w30)
    out["c_stack"], out["c_rF"], out["c_ru"], out["c_per_agent"] = w30, rep.r_F, rep.r_u, np.array(rep.per_agent)
    # (d) PnP with the identity denoiser: r_F and r_H
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.1, mode="pnp", denoiser=mt.DenoiserSpec(kind="identity"),
                           max_outer=10, tol=1e-300, residuals="none")
    w10 = fixed(mt.mace_pnp_solve, prob, cfg).stack
    rep = mt.mace.equilibrium_residuals(prob, cfg, w10)
    out["d_stack"], out["d_rF"], out["d_ru"], out["d_per_agent"] = w10, rep.r_F, rep.r_u, np.array(rep.per_agent)
    path = os.path.join(HERE, "golden_residuals.npz")
    np.savez_compressed(path, **out)
    for k in ("a", "b", "c", "d"):
        print(k, float(out[f"{k}_rF"]), float(out[f"{k}_ru"]))
    print("b iterations", out["b_iters"], "wrote", path)


if __name__ == "__main__":
    main()
