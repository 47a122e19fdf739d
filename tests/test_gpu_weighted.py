"""K2 weighted records (k_sv.cuh): slot records a sqrt(lambda) and the error sinogram kept as
sqrt(lambda) e give the same super-voxel iterates as the plain records with a lambda plane, the
error sinogram the host reads back is still y - A z, and data with a zero weight fall back to the
plain records."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import engine

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b)) / max(float(np.linalg.norm(b)), 1e-300)


def _ellipse_problem(golden):
    ns, nv, nc = 32, 45, 47
    geom = mb.Geometry(ns, 4.0, nv, nc, 4.0)
    return mb.ReconProblem(geom, mb.build_system_matrix(geom), golden["ell_y"], golden["ell_w"],
                           mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01))


def _solve(prob, weighted, iters, monkeypatch, sigma=3e-4, sv_side=4):
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    engine.clear_cache()
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=sigma, max_outer=iters, tol=1e-300, residuals="none",
                        schedule="sv", sv_side=sv_side)
    try:
        res = mb.mace_solve(prob, cfg)
    except mb.ConvergenceError as err:  # tol = 1e-300: a fixed iteration budget
        res = err.last_iterate
    views = [tuple(s.view_indices) for s in mb.partition_views(prob.geom.n_views, 4)]
    plan = engine.plan_for(prob.matrices, views, schedule="sv", sv=sv_side)
    flag = plan.info()["weighted"]
    engine.clear_cache()
    return res, flag


def test_weighted_and_plain_records_give_the_same_iterates(monkeypatch):
    # the setting of test_gpu_parity::test_sv_schedule_deterministic_enough_and_reproducible (a
    # strongly contracting iteration, where run-to-run float-atomic noise stays ~1e-6)
    ns, nv, nc = 8, 16, 11
    geom = mb.Geometry(ns, 1.0, nv, nc, ns / nc * 1.1)
    rng = np.random.default_rng(31)
    y = rng.standard_normal((nv, nc))
    w = 0.5 + rng.random((nv, nc))
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 1.0, sigma_x=0.5))
    rw, fw = _solve(prob, True, 50, monkeypatch, sigma=0.2, sv_side=8)
    rp, fp = _solve(prob, False, 50, monkeypatch, sigma=0.2, sv_side=8)
    assert (fw, fp) == (1, 0)
    assert rel(rw.image, rp.image) < 1e-5
    assert rel(rw.stack, rp.stack) < 1e-5


def test_weighted_fixed_point_is_the_centralized_map(golden, monkeypatch):
    prob = _ellipse_problem(golden)
    res, flag = _solve(prob, True, 3000, monkeypatch)
    assert flag == 1
    assert rel(res.image, golden["ell_central"]) < 1e-3


def test_weighted_error_sinogram_reads_back_as_residual(monkeypatch):
    monkeypatch.setenv("MACE_WEIGHTED", "1")
    ns, nv, nc = 16, 24, 23
    geom = mb.Geometry(ns, 1.0, nv, nc, 1.0)
    mats = mb.build_system_matrix(geom)
    rng = np.random.default_rng(4)
    y = rng.standard_normal((nv, nc))
    w = 0.5 + 100.0 * rng.random((nv, nc))  # wide weight range: sqrt(lambda) from 0.7 to 10
    prob = mb.ReconProblem(geom, mats, y, w, mb.PriorParams("qggmrf", 0.5, 2.0, 1.2, 1.0, 1.0))
    sub = mb.partition_views(nv, 2)[1]
    ws = mb.AgentWorkspace(prob, sub, 2, sigma=0.5, schedule="sv")
    assert ws.plan.info()["weighted"] == 1
    v = rng.standard_normal(ws.n)
    for _ in range(mb.REFRESH_EVERY + 3):
        mb.partial_update_prox(ws, v)
    assert ws.error_drift() < 1e-5
    # e read back = y_i - A_i z (icd.py:200), against the oracle's float64 forward projection
    ref_mats = O.build_system_matrix(ns, 1.0, nv, nc, 1.0)
    z = ws.state
    ax = O.forward_project(ref_mats, z)
    exact = np.concatenate([(y - ax)[j] for j in sub.view_indices])
    assert rel(ws.error_sinogram, exact) < 1e-5


def test_zero_weight_falls_back_to_plain_records(monkeypatch):
    monkeypatch.setenv("MACE_WEIGHTED", "1")
    ns, nv, nc = 16, 24, 23
    geom = mb.Geometry(ns, 1.0, nv, nc, 1.0)
    rng = np.random.default_rng(5)
    y = rng.standard_normal((nv, nc))
    w = 0.5 + rng.random((nv, nc))
    w[3, 5] = 0.0
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 0.5, 2.0, 1.2, 1.0, 1.0))
    sub = mb.partition_views(nv, 2)[0]
    a = mb.AgentWorkspace(prob, sub, 2, sigma=0.5, schedule="sv")
    b = mb.AgentWorkspace(prob, sub, 2, sigma=0.5, schedule="raster")
    assert a.plan.info()["weighted"] == 0
    v = rng.standard_normal(a.n)
    za = mb.prox_solve(a, v, tol=1e-7, max_passes=3000)
    zb = mb.prox_solve(b, v, tol=1e-7, max_passes=3000)
    assert rel(za, zb) < 1e-4


@pytest.mark.parametrize("sv_side", [2, 4, 6, 12, 16])
@pytest.mark.parametrize("weighted", [True, False])
def test_every_tile_side_reaches_the_raster_prox_point(sv_side, weighted, monkeypatch):
    """Every compiled tile side (k2_inst.cu units), with weighted and plain records: the parallel pass
    converges to the proximal point the reference-order raster pass reaches (icd.py:286-303).
    Sides 2 and 6 have parity classes that are not a multiple of four pixels (padding slots);
    a 30 x 30 image makes every side leave partial edge tiles."""
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    ns, nv, nc = 30, 36, 33
    geom = mb.Geometry(ns, 1.0, nv, nc, 1.0)
    rng = np.random.default_rng(40 + sv_side)
    y = rng.standard_normal((nv, nc))
    w = 0.5 + rng.random((nv, nc))
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 0.5, 2.0, 1.2, 1.0, 1.0))
    sub = mb.partition_views(nv, 3)[1]
    a = mb.AgentWorkspace(prob, sub, 3, sigma=0.5, schedule="raster")
    b = mb.AgentWorkspace(prob, sub, 3, sigma=0.5, schedule="sv", sv_side=sv_side)
    assert b.plan.info()["S"] == sv_side and b.plan.info()["weighted"] == int(weighted)
    v = rng.standard_normal(a.n)
    za = mb.prox_solve(a, v, tol=1e-7, max_passes=3000)
    zb = mb.prox_solve(b, v, tol=1e-7, max_passes=3000)
    assert rel(zb, za) < 1e-4


@pytest.mark.parametrize("sv_side", [4, 8])
@pytest.mark.parametrize("weighted", [True, False])
def test_sv_consts_theta2_matches_oracle(golden, sv_side, weighted, monkeypatch):
    """k_sv_consts (one block per tile, lambda window in shared memory): the theta2 image it writes
    per data load is sum_r a_r^2 lambda_r over each agent's rows (icd.py:193-195), for weighted and
    plain records, before and after a second data load with different weights."""
    prob = _ellipse_problem(golden)
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    engine.clear_cache()
    views = [tuple(s.view_indices) for s in mb.partition_views(prob.geom.n_views, 4)]
    plan = engine.plan_for(prob.matrices, views, schedule="sv", sv=sv_side)
    y = np.asarray(golden["ell_y"], np.float64)
    w0 = np.asarray(golden["ell_w"], np.float64)
    rng = np.random.default_rng(7)
    for w in (w0, w0 * rng.uniform(0.5, 2.0, size=w0.shape)):
        plan.load_data(y, w)
        assert bool(plan.info()["weighted"]) == weighted
        wv = w.reshape(prob.geom.n_views, -1)
        for i, vs in enumerate(views):
            import scipy.sparse as sp
            A = sp.vstack([O.view_csr(prob.matrices[v]) for v in vs]).tocsr()
            lam = np.concatenate([wv[v] for v in vs])
            ref = np.asarray(A.multiply(A).T @ lam).ravel()
            got = plan.get_theta2(i)
            assert rel(got, ref) < 1e-5, (i, rel(got, ref))
    engine.clear_cache()


def _slot_pixel(S, t):
    """internal.h sv_slot_pixel: visit-order slot t of an S x S tile -> local pixel, -1 for padding"""
    h = S // 2
    per_class = h * h
    bpc = (per_class + 3) // 4
    b, cls = t // 4, (t // 4) // bpc
    i = (b % bpc) * 4 + t % 4
    if i >= per_class:
        return -1
    return ((cls >> 1) + 2 * (i // h)) * S + (cls & 1) + 2 * (i % h)


@pytest.mark.parametrize("sv_side", [8, 16])
@pytest.mark.parametrize("weighted", [True, False])
def test_sv_consts_cross_terms_match_oracle(golden, sv_side, weighted, monkeypatch):
    """k_sv_consts' batch constants read back: for every batch of every tile, theta2 of
    the four slots and the six cross terms c_ij = sum_r a_ir a_jr lambda_r = (A^T diag(lambda) A)[p_i, p_j]
    against the oracle CSR, tile sides 8 and 16 (16 and 64 batches per tile, so the next-batch
    prefetch runs for every warp), weighted and plain records."""
    import scipy.sparse as sp

    prob = _ellipse_problem(golden)
    monkeypatch.setenv("MACE_WEIGHTED", "1" if weighted else "0")
    engine.clear_cache()
    views = [tuple(s.view_indices) for s in mb.partition_views(prob.geom.n_views, 4)]
    plan = engine.plan_for(prob.matrices, views, schedule="sv", sv=sv_side)
    plan.load_data(golden["ell_y"], golden["ell_w"])
    assert bool(plan.info()["weighted"]) == weighted
    ns = prob.geom.n_side
    wv = np.asarray(golden["ell_w"], np.float64).reshape(prob.geom.n_views, -1)
    nss = -(-ns // sv_side)
    pairs = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    checked = 0
    for i, vs in enumerate(views[:2]):
        A = sp.vstack([O.view_csr(prob.matrices[v]) for v in vs]).tocsc()
        lam = np.concatenate([wv[v] for v in vs])
        M = (A.T @ sp.diags(lam) @ A).tocsr()  # n x n, exact in float64
        bc = plan.get_batch_consts(i)
        assert bc.shape[0] == nss * nss
        for sv in range(bc.shape[0]):
            r0, c0 = (sv // nss) * sv_side, (sv % nss) * sv_side
            for b in range(bc.shape[1]):
                px = []
                for p in range(4):
                    k = _slot_pixel(sv_side, 4 * b + p)
                    r, c = (r0 + k // sv_side, c0 + k % sv_side) if k >= 0 else (ns, ns)
                    px.append(r * ns + c if (r < ns and c < ns) else -1)
                ref = np.zeros(10)
                for p in range(4):
                    if px[p] >= 0:
                        ref[p] = M[px[p], px[p]]
                for j, (p, q) in enumerate(pairs):
                    if px[p] >= 0 and px[q] >= 0:
                        ref[4 + j] = M[px[p], px[q]]
                got = bc[sv, b, :10].astype(np.float64)
                scale = max(np.abs(ref[:4]).max(), 1e-30)
                assert np.abs(got - ref).max() <= 1e-5 * scale, (sv, b, got, ref)
                checked += 1
    print(f"sv {sv_side} weighted {weighted}: {checked} batches checked")
    engine.clear_cache()
