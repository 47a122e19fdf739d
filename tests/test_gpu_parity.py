"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden vectors.  Tolerances (fp32 device arithmetic vs fp64 reference):

* raster schedule (reference visiting order): 1e-5 relative per pass / per iterate;
* super-voxel schedule (parallel, different order, same fixed point): the
  converged image within relative RMSE 1e-3 of the converged reference (BASELINE.json).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import small_problem

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b)) / max(float(np.linalg.norm(b)), 1e-300)


def mb_problem(seed, ns, nv, nc, kind, beta, sx):
    mats = mb.build_system_matrix(mb.Geometry(ns, 1.0, nv, nc, ns / nc * 1.1))
    _, y, w = small_problem(seed, ns, nv, nc)
    return mb.ReconProblem(mb.Geometry(ns, 1.0, nv, nc, ns / nc * 1.1), mats, y, w,
                           mb.PriorParams(kind=kind, beta=beta, sigma_x=sx))


CASES = ["pq", "pg", "pg2", "pq2", "pg3"]


def _ws_from_golden(g, name, schedule="raster"):
    seed, ns, nv, nc, beta, sx, N, agent, sigma, is_qg = g[f"{name}_meta"]
    prob = mb_problem(int(seed), int(ns), int(nv), int(nc), "qggmrf" if is_qg else "quadratic-mrf", float(beta),
                      float(sx))
    sub = mb.partition_views(int(nv), int(N))[int(agent)]
    return mb.AgentWorkspace(prob, sub, int(N), sigma=float(sigma), state=g[f"{name}_x0"], schedule=schedule)


@pytest.mark.parametrize("name", CASES)
def test_raster_pass_matches_reference_per_pass(golden, name):
    ws = _ws_from_golden(golden, name)
    assert rel(ws.curv_data, golden[f"{name}_curv"]) < 1e-6
    assert rel(ws.error_sinogram, golden[f"{name}_e0"]) < 1e-6
    v = golden[f"{name}_v"]
    z1 = mb.partial_update_prox(ws, v)
    assert rel(z1, golden[f"{name}_z1"]) < 1e-5
    assert rel(ws.error_sinogram, golden[f"{name}_e1"]) < 1e-5
    for _ in range(4):
        z5 = mb.partial_update_prox(ws, v)
    assert rel(z5, golden[f"{name}_z5"]) < 1e-5


@pytest.mark.parametrize("name", CASES)
def test_pixel_update_matches_reference(golden, name):
    ws = _ws_from_golden(golden, name)
    s = min(7, ws.n - 1)
    alpha = mb.pixel_update(ws, s, golden[f"{name}_v"])
    assert alpha == pytest.approx(golden[f"{name}_alpha7"][0], rel=1e-4, abs=1e-6)


@pytest.mark.parametrize("name", CASES)
def test_sv_schedule_prox_fixed_point_matches_raster(golden, name):
    """Different visiting order, same proximal point (icd.py:286-303)."""
    a = _ws_from_golden(golden, name, "raster")
    b = _ws_from_golden(golden, name, "sv")
    v = golden[f"{name}_v"]
    za = mb.prox_solve(a, v, tol=1e-6, max_passes=2000)
    zb = mb.prox_solve(b, v, tol=1e-6, max_passes=2000)
    assert rel(zb, za) < 1e-4


def _zero_cost_ws(sigma=1.0, schedule="raster"):
    geom = mb.Geometry(4, 1.0, 2, 3, 1.0)
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), np.zeros((2, 3)), np.zeros((2, 3)),
                           mb.PriorParams(beta=0.0))
    return mb.AgentWorkspace(prob, mb.partition_views(2, 1)[0], 1, sigma=sigma, schedule=schedule)


@pytest.mark.parametrize("schedule", ["raster", "sv"])
def test_zero_cost_pass_returns_target(schedule):
    ws = _zero_cost_ws(schedule=schedule)
    v = np.random.default_rng(1).standard_normal(ws.n)
    out = mb.partial_update_prox(ws, v)
    assert np.allclose(out, v.astype(np.float32), rtol=2e-7, atol=0)


def test_scalar_kat_alpha_one():
    geom = mb.Geometry(1, 1.0, 1, 1, 1.0)
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), np.zeros((1, 1)), np.ones((1, 1)),
                           mb.PriorParams(beta=0.0))
    ws = mb.AgentWorkspace(prob, mb.partition_views(1, 1)[0], 1, sigma=1.0)
    assert mb.pixel_update(ws, 0, np.array([2.0])) == pytest.approx(1.0, rel=1e-6)


def test_error_sinogram_drift_and_refresh():
    prob = mb_problem(71, 6, 12, 9, "quadratic-mrf", 0.5, 1.0)
    ws = mb.AgentWorkspace(prob, mb.partition_views(12, 2)[1], 2, sigma=0.5)
    v = np.random.default_rng(10).standard_normal(ws.n)
    for _ in range(mb.REFRESH_EVERY + 5):
        mb.partial_update_prox(ws, v)
    assert ws.error_drift() < 1e-5
    assert ws.passes == mb.REFRESH_EVERY + 5


def test_forward_project_and_cost_vs_oracle(golden):
    ns, pp, nv, nc, cp = 32, 4.0, 64, 47, 4.0
    mats = mb.build_system_matrix(mb.Geometry(ns, pp, nv, nc, cp))
    x = np.random.default_rng(3).random(ns * ns) * 0.05
    fp = mb.forward_project(mats, x)
    ref = O.forward_project(mats, x)
    assert np.max(np.abs(fp - ref)) / np.max(np.abs(ref)) < 1e-5
    assert rel(fp, ref) < 1e-5
    y, lam = gen.poisson_sinogram(ref, 1e4, seed=2)
    prob = mb.ReconProblem(mb.Geometry(ns, pp, nv, nc, cp), mats, y, lam,
                           mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01))
    c = mb.map_cost(prob, x)
    c_ref = O.likelihood_cost(mats, y, lam, x) + O.prior_cost(x, "qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01, 0, ns)
    assert c == pytest.approx(c_ref, rel=1e-5)


def _mq_problem(golden):
    prob = mb_problem(31, 8, 16, 11, "qggmrf", 1.0, 0.5)
    assert np.array_equal(prob.y, golden["mq_y"])
    return prob


def _fixed(fn, *a, **k):
    try:
        return fn(*a, **k)
    except mb.ConvergenceError as err:
        return err.last_iterate


def test_mace_raster_fixed_budget_matches_reference(golden):
    prob = _mq_problem(golden)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=12, tol=1e-300, residuals="none",
                        schedule="raster")
    res = _fixed(mb.mace_solve, prob, cfg)
    assert res.iterations == 12
    assert rel(res.stack, golden["mq_stack"]) < 1e-5
    assert rel(res.image, golden["mq_image"]) < 1e-5
    relnorm = np.array([r["relnorm"] for r in res.log.rows])
    assert np.allclose(relnorm, golden["mq_relnorm"], rtol=1e-3)


@pytest.mark.parametrize("schedule", ["raster", "sv"])
def test_mace_converges_to_centralized_map(golden, schedule):
    """MACE fixed point = centralized MAP; oracle = reference icd_map_solve."""
    prob = _mq_problem(golden)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=20000, tol=1e-7, residuals="none",
                        schedule=schedule)
    res = mb.mace_solve(prob, cfg)
    assert res.converged
    assert rel(res.image, golden["mq_central"]) < 1e-3


def test_mace_counts_weighted_ellipse_fixed_point(golden):
    """Miniature of the benchmark recipe (counts weights, qGGMRF p=2 q=1.2, sigma_x=0.01)."""
    ns, nv, nc = 32, 45, 47
    geom = mb.Geometry(ns, 4.0, nv, nc, 4.0)
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), golden["ell_y"], golden["ell_w"],
                           mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01))
    cfg30 = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=3e-4, max_outer=30, tol=1e-300, residuals="none",
                          schedule="raster")
    r30 = _fixed(mb.mace_solve, prob, cfg30)
    assert rel(r30.image, golden["ell_image30"]) < 1e-4
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=3e-4, max_outer=3000, tol=1e-300, residuals="none",
                        schedule="sv", sv_side=4)
    res = _fixed(mb.mace_solve, prob, cfg, ref_image=golden["ell_central"])
    nr = [r["nrmse"] for r in res.log.rows]
    assert nr[-1] < 1e-3
    assert mb.map_cost(prob, res.image) == pytest.approx(golden["ell_cost_central"][0], rel=1e-4)


def _boxcar(n_side):
    def H(v):
        m = n_side
        img = np.asarray(v, np.float64).reshape(m, m)
        sat = np.zeros((m + 1, m + 1))
        sat[1:, 1:] = np.cumsum(np.cumsum(img, axis=0), axis=1)
        i = np.arange(m)
        lo, hi = np.maximum(i - 1, 0), np.minimum(i + 2, m)
        box = sat[np.ix_(hi, hi)] - sat[np.ix_(lo, hi)] - sat[np.ix_(hi, lo)] + sat[np.ix_(lo, lo)]
        return (box / np.outer(hi - lo, hi - lo)).ravel()
    return H


def test_mace_pnp_custom_callable_matches_reference(golden):
    prob = _mq_problem(golden)
    calls = []

    def H(v):
        calls.append(1)
        return _boxcar(8)(v)

    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.1, mode="pnp", denoiser=mb.DenoiserSpec("identity"),
                        max_outer=10, tol=1e-300, residuals="none", schedule="raster")
    res = _fixed(mb.mace_pnp_solve, prob, cfg, denoiser=H)
    assert calls
    assert rel(res.stack, golden["mp_stack"]) < 1e-5
    assert rel(res.image, golden["mp_image"]) < 1e-5


def test_mace_divergence_detected():
    prob = mb_problem(2, 6, 12, 9, "quadratic-mrf", 0.5, 1.0)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=50.0, tol=1e-9, max_outer=100000, residuals="none")
    with pytest.raises(mb.ConvergenceError, match="diverged|relnorm"):
        mb.mace_solve(prob, cfg)


def test_warm_start_is_stationary(golden):
    prob = _mq_problem(golden)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=20000, tol=1e-7, residuals="none",
                        schedule="raster")
    res = mb.mace_solve(prob, cfg)
    res2 = mb.mace_solve(prob, cfg, w0=res.stack)
    assert res2.log.rows[0]["relnorm"] < 1e-5


def test_sv_schedule_deterministic_enough_and_reproducible(golden):
    prob = _mq_problem(golden)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=50, tol=1e-300, residuals="none")
    a = _fixed(mb.mace_solve, prob, cfg).image
    b = _fixed(mb.mace_solve, prob, cfg).image
    assert rel(a, b) < 1e-5


def test_errors_and_validation(golden):
    prob = _mq_problem(golden)
    with pytest.raises(ValueError):
        mb.mace_solve(prob, mb.MaceConfig(n_subsets=2, mode="pnp", denoiser=mb.DenoiserSpec("identity")))
    with pytest.raises(ValueError):
        mb.mace_pnp_solve(prob, mb.MaceConfig(n_subsets=2))
    with pytest.raises(ValueError):
        mb.mace_solve(prob, mb.MaceConfig(n_subsets=4, residuals="none"), w0=np.zeros((3, prob.n)))
    sub = mb.partition_views(16, 1)[0]
    with pytest.raises(ValueError):
        mb.AgentWorkspace(prob, sub, 1, sigma=0.0)
    ws = mb.AgentWorkspace(prob, sub, 1, sigma=1.0)
    with pytest.raises(ValueError):
        mb.pixel_update(ws, prob.n, np.zeros(prob.n))
    with pytest.raises(ValueError):
        mb.partial_update_prox(ws, np.zeros(prob.n - 1))
    with pytest.raises(ValueError):
        mb.prox_solve(ws, np.zeros(prob.n), tol=0.0)


def test_agents_with_many_views():
    """More than 128 views per agent: the super-voxel schedule runs multi-warp tiles (two 96-view
    chunks per 150-view agent, tests/test_gpu_multiwarp.py), and the raster schedule stays iterate
    for iterate equal to the oracle's MACE: 2 agents x 150 views, ragged 37 x 37 image."""
    ns, nv, nc = 37, 300, 41
    geom = mb.Geometry(ns, 1.0, nv, nc, 1.0)
    mats = mb.build_system_matrix(geom)
    ph = np.zeros(ns * ns)
    ph[(np.arange(ns * ns) % 7) == 0] = 0.02
    y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 1e4, seed=9)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", 50.0, 2.0, 1.2, 1.0, 0.01))
    plan = mb.engine.plan_for(mats, [s.view_indices for s in mb.partition_views(nv, 2)], schedule="sv")
    assert plan.schedule == "sv" and plan.info()["n_items"] == 2 * 5 * 5
    iters, sigma = 25, 1e-4
    cfg = mb.MaceConfig(n_subsets=2, rho=0.8, sigma=sigma, max_outer=iters, tol=1e-300, residuals="none",
                        schedule="raster")
    res = _fixed(mb.mace_solve, prob, cfg)
    agents = O.build_agents(mats, y, lam, 2, sigma, O.Prior("qggmrf", 50.0, 2.0, 1.2, 1.0, 0.01), ns)
    run = O.mace_run(agents, iters, 0.8)
    assert rel(res.image, run.image) < 1e-4


def _clamp_problem():
    """Low-count scan of a sparse phantom: the unconstrained iterates go negative in the background,
    so the non-negativity clamp (icd.py:130-134, clamp_nonneg) is active on many pixels."""
    ns, nv, nc = 32, 45, 47
    pitch = 4.0
    geom = mb.Geometry(ns, pitch, nv, nc, pitch)
    mats = mb.build_system_matrix(geom)
    ph = gen.ellipse_phantom(ns, pitch, 3, seed=21) * 0.3
    y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 300.0, seed=22)
    prior = mb.PriorParams("qggmrf", 5.0, 2.0, 1.2, 1.0, 0.01)
    return geom, mats, y, lam, mb.ReconProblem(geom, mats, y, lam, prior), O.Prior("qggmrf", 5.0, 2.0, 1.2, 1.0, 0.01)


def test_clamped_mace_raster_matches_oracle():
    geom, mats, y, lam, prob, oprior = _clamp_problem()
    iters, sigma, N = 80, 3e-4, 4
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=sigma, max_outer=iters, tol=1e-300, residuals="none",
                        schedule="raster", clamp_nonneg=True)
    res = _fixed(mb.mace_solve, prob, cfg)
    run = O.mace_run(O.build_agents(mats, y, lam, N, sigma, oprior, geom.n_side, clamp=True), iters, 0.8)
    assert rel(res.image, run.image) < 1e-4
    free = O.mace_run(O.build_agents(mats, y, lam, N, sigma, oprior, geom.n_side), iters, 0.8)
    assert free.image.min() < -1e-4  # the clamp was active


def test_clamped_mace_sv_reaches_the_clamped_map():
    """super-voxel schedule (4-pixel batches, clamp inside the exact in-batch recurrence) converges to
    the fixed point of the clamped centralized ICD"""
    geom, mats, y, lam, prob, oprior = _clamp_problem()
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=3e-4, max_outer=10000, tol=1e-300, residuals="none",
                        schedule="sv", sv_side=4, clamp_nonneg=True)
    res = _fixed(mb.mace_solve, prob, cfg)
    ag = O.Agent(mats, y, lam, range(geom.n_views), 1, None, oprior, geom.n_side, clamp=True)
    v = np.zeros(ag.n)
    for _ in range(5000):
        dsq = ag.run_range(v, 0, ag.n)
        if np.sqrt(dsq) < 1e-11 * max(np.linalg.norm(ag.state), 1e-300):
            break
    assert ag.state.min() >= 0.0
    assert res.image.min() >= -1e-9  # the consensus average of the stack, non-negative up to rounding
    assert rel(res.image, ag.state) < 2e-3


@pytest.mark.parametrize("case", ["mq", "ell"])
def test_icd_map_solve_matches_reference_central(golden, case):
    """Centralized ICD on the GPU (icd.py:306-345: one agent with every view, no proximal term,
    raster passes until sqrt(sum alpha^2)/||z|| < tol) against the reference's own
    icd_map_solve (golden mq_central at tol 1e-12, ell_central at 1e-11).  float32 state: tol
    1e-6, then the image within 1e-4 of the reference's."""
    if case == "mq":
        prob = _mq_problem(golden)
    else:
        geom = mb.Geometry(32, 4.0, 45, 47, 4.0)
        prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), golden["ell_y"], golden["ell_w"],
                               mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01))
    passes = []
    x = mb.icd_map_solve(prob, tol=1e-6, max_passes=5000, on_pass=lambda k, r, z: passes.append(r))
    err = rel(x, golden[f"{case}_central"])
    print(f"icd_map_solve {case}: {len(passes)} passes to 1e-6, NRMSE vs the reference's MAP {err:.2e}")
    assert err < 1e-4
    counter = mb.EquitCounter(prob.geom.n_pixels, 1)
    mb.icd_map_solve(prob, tol=1e-3, counter=counter)
    assert counter.equits() >= 1
    with pytest.raises(mb.ConvergenceError):
        mb.icd_map_solve(prob, tol=1e-12, max_passes=3)


def test_raster_schedule_is_bitwise_deterministic(golden):
    """The deterministic option: the raster schedule (reference visiting order, no atomics) gives
    bit-identical iterates run to run, as the reference does for a fixed worker count
    (tests/test_mace.py:161-170 of the reference); the super-voxel schedule agrees to ~1e-6."""
    prob = _mq_problem(golden)
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=60, tol=1e-300, residuals="none",
                        schedule="raster")
    a, b = _fixed(mb.mace_solve, prob, cfg), _fixed(mb.mace_solve, prob, cfg)
    assert np.array_equal(a.image, b.image) and np.array_equal(a.stack, b.stack)
    assert [r["relnorm"] for r in a.log.rows] == [r["relnorm"] for r in b.log.rows]


@pytest.mark.parametrize("n", [1, 4])
def test_mace_pnp_builtin_quadratic_prox_matches_reference(n):
    """MACE-PnP with the reference's built-in quadratic-prox denoiser (DenoiserSpec, applied on the
    host once per iteration as the reference does) at one and four agents lands on the reference's
    own fixed points (tests/golden/golden_denoisers.npz, made by make_denoisers.py; the reference's
    test_mace.py:298-306 asserts they coincide)."""
    import os

    from conftest import GOLDEN

    dg = np.load(os.path.join(GOLDEN, "golden_denoisers.npz"))
    prob = mb_problem(31, 8, 16, 11, "qggmrf", 1.0, 0.5)
    assert np.array_equal(prob.y, dg["pnp_y"])
    cfg = mb.MaceConfig(n_subsets=n, rho=0.8, sigma=0.1, mode="pnp",
                        denoiser=mb.DenoiserSpec(kind="quadratic-prox", lam=2.0), tol=1e-300, max_outer=4000,
                        residuals="none", schedule="raster")
    res = _fixed(mb.mace_pnp_solve, prob, cfg)  # fp32 state: a fixed budget instead of tol 1e-11
    assert res.iterations == 4000
    for k in (1, 4):
        assert rel(res.image, dg[f"pnp_image_n{k}"]) < 1e-5
