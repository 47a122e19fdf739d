"""Config 3 at full size (MACE-PnP, 512^2, 720 x 725, N = 8, BASELINE's 17-layer CNN, K5 on the
tensor cores inside the device loop) against the CPU oracle.

* raster schedule (the reference's visiting order, one warp per agent): 40 iterations from
  w = 0 must land within 1e-4 NRMSE of the oracle's own 40 iterations
  (tests/golden/pnp_c3_raster40.npz: oracle.mace_run, float64 raster agents, the torch CPU
  CNN; make_pnp_c3.py);
* super-voxel schedule (the bench's) against the raster schedule: both are Mann iterations of
  maps with the same fixed point, so from the super-voxel state after 3,000 iterations one
  raster iteration moves the stack by no more than a small multiple of what one more
  super-voxel iteration moves it (far from a fixed point of the raster map the step would be
  orders of magnitude larger)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen
from paper_1911_09278_b200.denoisers import CnnDenoiser

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    c = gen.CONFIGS[3]
    geom, mats, _, y, lam = gen.make_scan(3)
    prior = mb.PriorParams("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01)
    return c, mb.ReconProblem(geom, mats, y, lam, prior), CnnDenoiser(geom.n_side, seed=0)


def _cfg(c, iters, schedule):
    return mb.MaceConfig(n_subsets=c["n_agents"], rho=0.8, sigma=c["sigma"], mode="pnp",
                         denoiser=mb.DenoiserSpec("identity"), max_outer=iters, tol=1e-300, residuals="none",
                         schedule=schedule)


def _solve(prob, cfg, H, w0=None):
    try:
        return mb.mace_pnp_solve(prob, cfg, denoiser=H, w0=w0)
    except mb.ConvergenceError as err:
        return err.last_iterate


def test_pnp_raster_40_iterations_match_oracle(c3):
    c, prob, H = c3
    ref = np.load(os.path.join(GOLDEN, "pnp_c3_raster40.npz"))
    res = _solve(prob, _cfg(c, 40, "raster"), H)
    assert res.iterations == 40
    x_ref = ref["image"].astype(np.float64)
    err = float(np.linalg.norm(res.image - x_ref) / np.linalg.norm(x_ref))
    rel = np.array([r["relnorm"] for r in res.log.rows])
    print(f"config 3 raster, 40 iterations: NRMSE vs oracle {err:.2e}; relnorm {rel[-1]:.3e} "
          f"(oracle {float(ref['relnorm'][-1]):.3e})")
    assert err <= 1e-4
    assert np.allclose(rel, ref["relnorm"], rtol=1e-3)


def test_pnp_sv_state_is_near_raster_fixed_point(c3):
    c, prob, H = c3
    sv = _solve(prob, _cfg(c, 3000, "sv"), H)
    rel_sv = sv.log.rows[-1]["relnorm"]
    ra = _solve(prob, _cfg(c, 1, "raster"), H, w0=sv.stack)
    rel_ra = ra.log.rows[-1]["relnorm"]
    moved = float(np.linalg.norm(ra.image - sv.image) / np.linalg.norm(sv.image))
    print(f"config 3: super-voxel relnorm after 3000 iterations {rel_sv:.3e}; one raster iteration from "
          f"that stack: relnorm {rel_ra:.3e}, image moved {moved:.2e}")
    assert rel_ra <= 10 * rel_sv
    assert moved <= 1e-3
