"""K2 multi-warp tiles (k_sv.cuh, MW > 0): agents with more than 128 views -- the centralized ICD
of icd_map_solve (icd.py:306-345) and MACE with few agents -- run the parallel super-voxel pass
with one warp per chunk of 96 views of a tile.  The chunked batch constants are checked against
the oracle CSR, the pass against the reference-order raster pass's proximal point, and the
centralized solve against the CPU oracle's MAP (config 0 at full size: 180 views, 2 chunks)."""

from __future__ import annotations

import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import engine, gen

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b)) / max(float(np.linalg.norm(b)), 1e-300)


def _many_view_problem(nv, seed=3, ns=24, nc=27):
    geom = mb.Geometry(ns, 1.0, nv, nc, 1.0)
    rng = np.random.default_rng(seed)
    y = rng.standard_normal((nv, nc))
    w = 0.5 + rng.random((nv, nc))
    return mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 0.5, 2.0, 1.2, 1.0, 1.0))


def _slot_pixel(S, t):
    h = S // 2
    per_class = h * h
    bpc = (per_class + 3) // 4
    b, cls = t // 4, (t // 4) // bpc
    i = (b % bpc) * 4 + t % 4
    if i >= per_class:
        return -1
    return ((cls >> 1) + 2 * (i // h)) * S + (cls & 1) + 2 * (i % h)


@pytest.mark.parametrize("nv", [200, 1000])
@pytest.mark.parametrize("weighted", [True, False])
def test_chunked_batch_constants_match_oracle(nv, weighted, monkeypatch):
    """theta2 and the six cross terms of every batch, summed over all chunks' views, against
    (A^T diag(lambda) A) from the oracle CSR: 200 views = 7 groups -> 3 chunks; 1000 views = 32
    groups -> 11 chunks (the 512-thread instantiation)."""
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    engine.clear_cache()
    prob = _many_view_problem(nv)
    S = 8
    views = [tuple(range(nv))]
    plan = engine.plan_for(prob.matrices, views, schedule="sv", sv=S)
    assert plan.schedule == "sv"
    plan.load_data(prob.y, prob.weights)
    assert bool(plan.info()["weighted"]) == weighted
    A = sp.vstack([O.view_csr(prob.matrices[v]) for v in range(nv)]).tocsc()
    lam = np.asarray(prob.weights, np.float64).ravel()
    M = (A.T @ sp.diags(lam) @ A).tocsr()
    assert rel(plan.get_theta2(0), M.diagonal()) < 1e-5
    ns = prob.geom.n_side
    nss = -(-ns // S)
    bc = plan.get_batch_consts(0)
    pairs = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    for sv in range(nss * nss):
        r0, c0 = (sv // nss) * S, (sv % nss) * S
        for b in range(bc.shape[1]):
            px = []
            for p in range(4):
                k = _slot_pixel(S, 4 * b + p)
                r, c = (r0 + k // S, c0 + k % S) if k >= 0 else (ns, ns)
                px.append(r * ns + c if (r < ns and c < ns) else -1)
            for p in range(4):
                if px[p] >= 0:
                    assert bc[sv, b, p] == pytest.approx(M[px[p], px[p]], rel=2e-5, abs=1e-6)
            for x, (i, j) in enumerate(pairs):
                if px[i] >= 0 and px[j] >= 0:
                    assert bc[sv, b, 4 + x] == pytest.approx(M[px[i], px[j]], rel=2e-5, abs=1e-5 * M[px[i], px[i]])
    engine.clear_cache()


@pytest.mark.parametrize("nv", [150, 300])
@pytest.mark.parametrize("weighted", [True, False])
def test_multiwarp_pass_reaches_the_raster_prox_point(nv, weighted, monkeypatch):
    """One agent with every view (150 -> 2 chunks, 300 -> 4 chunks): the multi-warp super-voxel
    pass converges to the proximal point of the reference-order raster pass (icd.py:286-303)."""
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    engine.clear_cache()
    prob = _many_view_problem(nv, seed=nv)
    sub = mb.ViewSubset(0, tuple(range(nv)))
    a = mb.AgentWorkspace(prob, sub, 1, sigma=0.5, schedule="raster")
    b = mb.AgentWorkspace(prob, sub, 1, sigma=0.5, schedule="sv", sv_side=8)
    assert b.plan.schedule == "sv" and b.plan.info()["weighted"] == int(weighted)
    v = np.random.default_rng(nv).standard_normal(a.n)
    za = mb.prox_solve(a, v, tol=1e-7, max_passes=3000)
    zb = mb.prox_solve(b, v, tol=1e-7, max_passes=3000)
    assert rel(zb, za) < 1e-4
    # the error sinogram stays consistent with the state (every chunk's rows were written back)
    e = b.error_sinogram
    b.refresh_error()
    assert rel(e, b.error_sinogram) < 1e-5
    engine.clear_cache()


def _central_sv(config, passes):
    """icd_map_solve on the super-voxel schedule (proximal-anchored parallel passes, icd.py
    CENTRAL_KAPPA) for a fixed pass budget (tol below the fp32 / float-atomic floor of relnorm, so
    the solve runs `passes` passes and raises with its iterate)."""
    import time

    c = gen.CONFIGS[config]
    geom, mats, phantom, y, lam = gen.make_scan(config)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01))
    rn = []
    t0 = time.perf_counter()
    with pytest.raises(mb.ConvergenceError) as ei:
        mb.icd_map_solve(prob, tol=1e-30, max_passes=passes, schedule="sv", on_pass=lambda k, r, z: rn.append(r))
    dt = time.perf_counter() - t0
    engine.clear_cache()
    return np.asarray(ei.value.last_iterate, np.float64), np.asarray(rn), dt


def test_icd_map_solve_multiwarp_matches_cpu_oracle_map_c0():
    """Config 0 at full size (128^2, 180 views: 2 chunks per tile): the centralized solve on the
    parallel multi-warp pass lands on the CPU oracle's float64 MAP (tests/golden/central_c0.npz)."""
    ref = np.load(os.path.join(GOLDEN, "central_c0.npz"))["image"]
    x, rn, dt = _central_sv(0, 600)
    err = rel(x, ref)
    print(f"icd_map_solve c0 (sv, 2 chunks): 600 passes in {dt:.2f} s, relnorm {rn[99]:.1e} @100 "
          f"{rn[299]:.1e} @300 {rn[-1]:.1e} @600, NRMSE vs oracle MAP {err:.2e}")
    assert err < 1e-4
    assert rn[-1] < 1e-4 * rn[0]


def test_icd_map_solve_multiwarp_matches_cpu_oracle_map_c1():
    """Config 1 at full size (512^2, 720 views: 8 chunks per tile, the c1 centralized problem)
    against the CPU oracle's MAP (tests/golden/central_c1.npz, tol 1e-7)."""
    ref = np.load(os.path.join(GOLDEN, "central_c1.npz"))["image"]
    x, rn, dt = _central_sv(1, 600)
    err = rel(x, ref)
    print(f"icd_map_solve c1 (sv, 8 chunks): 600 passes in {dt:.2f} s (incl. setup), relnorm {rn[99]:.1e} @100 "
          f"{rn[299]:.1e} @300 {rn[-1]:.1e} @600, NRMSE vs oracle MAP {err:.2e}")
    assert err < 2e-4


def test_mace_one_agent_many_views_fixed_point():
    """MACE with a single agent owning all 180 views of config 0 (a multi-warp K2 inside the device
    loop): the fixed point is the centralized MAP."""
    ref = np.load(os.path.join(GOLDEN, "central_c0.npz"))["image"]
    c = gen.CONFIGS[0]
    geom, mats, phantom, y, lam = gen.make_scan(0)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", c["beta"], 2.0, 1.2, 1.0, 0.01))
    cfg = mb.MaceConfig(n_subsets=1, rho=0.8, sigma=c["sigma"], max_outer=3000, tol=1e-300, residuals="none",
                        schedule="sv")
    try:
        res = mb.mace_solve(prob, cfg)
    except mb.ConvergenceError as err:
        res = err.last_iterate
    err = rel(res.image, ref)
    print(f"MACE N=1 (180 views, multi-warp) after 3000 iterations: NRMSE vs oracle MAP {err:.2e}")
    assert err < 1e-3
    engine.clear_cache()
