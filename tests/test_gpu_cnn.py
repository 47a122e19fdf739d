"""K5 (tcgen05 implicit-GEMM CNN denoiser) against the torch CPU oracle (oracle/cnn.py),
and MACE-PnP with it (BASELINE config 3 recipe) against the oracle loop with the same
callable.

Tolerances: the GPU accumulates in fp32 and both sides round activations to bf16 between
layers, so an activation can land one bf16 ulp (2^-8 relative) apart when the fp32 sum
straddles a rounding boundary.  The residual net(x) is checked to 2e-2 relative (L2) and the
denoised image x - net(x) to 1e-4 relative."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from cnn import cnn_apply

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen
from paper_1911_09278_b200.denoisers import CnnDenoiser, cnn_weights

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n_side,seed", [(64, 0), (512, 1), (200, 2), (130, 3)])
def test_cnn_matches_cpu_oracle(n_side, seed):
    rng = np.random.default_rng(seed)
    x = 0.02 + 0.01 * rng.standard_normal(n_side * n_side)
    w = cnn_weights(seed)
    H = CnnDenoiser(n_side, weights=w)
    out = H(x)
    ref = cnn_apply(x, w, n_side)
    assert rel(x - out, x - ref) < 2e-2, rel(x - out, x - ref)
    assert rel(out, ref) < 1e-4
    print(f"n={n_side}: K5 {H.last_ms:.3f} ms, residual rel err {rel(x - out, x - ref):.2e}")


def test_cnn_non_trivial_weights():
    """Unit-scale weights (no 0.1 factor): the net output is O(x), so the check is not vacuous."""
    n = 128
    rng = np.random.default_rng(7)
    x = rng.random(n * n)
    w = cnn_weights(5, scale=1.0)
    out = CnnDenoiser(n, weights=w)(x)
    ref = cnn_apply(x, w, n)
    assert rel(x - ref, x) > 0.05
    assert rel(x - out, x - ref) < 2e-2


def test_mace_pnp_with_cnn_denoiser_vs_oracle_loop():
    """Config-3 recipe in miniature: PnP agents at sqrt(N) sigma, beta = 0, H = the CNN."""
    ns, nv, nc, N = 64, 90, 91, 4
    pitch = 128.0 / ns
    geom = mb.Geometry(ns, pitch, nv, nc, pitch)
    mats = mb.build_system_matrix(geom)
    ph = gen.ellipse_phantom(ns, pitch, 10, seed=0)
    y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 1e4, seed=1)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", 25.0, 2.0, 1.2, 1.0, 0.01))
    w = cnn_weights(3)
    H = CnnDenoiser(ns, weights=w)
    sigma, iters = 2e-4, 20
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=sigma, mode="pnp", denoiser=mb.DenoiserSpec("identity"),
                        max_outer=iters, tol=1e-300, residuals="none", schedule="raster")
    try:
        res = mb.mace_pnp_solve(prob, cfg, denoiser=H)
    except mb.ConvergenceError as err:
        res = err.last_iterate
    agents = O.build_agents(mats, y, lam, N, sigma, O.Prior("qggmrf", 25.0, 2.0, 1.2, 1.0, 0.01), ns, pnp=True)
    run = O.mace_run(agents, iters, 0.8, denoiser=lambda v: cnn_apply(v, w, ns))
    assert rel(res.image, run.image) < 1e-4
