"""MAP-cost gradient (mace_gradient): against a float64 numpy restatement of the reference cost
model (models.py:235-278, oracle/oracle.py), and ~0 at the converged oracle MAP (the certificate
used where no CPU oracle can be converged)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

import paper_1911_09278_b200 as mb

pytestmark = pytest.mark.gpu


def _np_gradient(mats, y, lam, x, kind, beta, p, q, T, sx, eps, n_side):
    g = np.zeros(n_side * n_side)
    for k, m in enumerate(mats):
        A = O.view_csr(m)
        g -= A.T @ (lam[k] * (y[k] - A @ x))
    idx, w = O.neighbor_table(n_side)
    d = x[:, None] - np.where(idx >= 0, x[np.maximum(idx, 0)], 0.0)
    infl = d if kind == "quadratic-mrf" else O.qggmrf_influence(d, p, q, T, sx)
    gp = np.sum(w * infl, axis=1)
    if kind == "quadratic-mrf":
        gp += 2.0 * eps * x
    return g + beta * gp


@pytest.mark.parametrize("kind", ["qggmrf", "quadratic-mrf"])
def test_gradient_matches_numpy(golden, kind):
    ns, nv, nc = 32, 45, 47
    geom = mb.Geometry(ns, 4.0, nv, nc, 4.0)
    mats = mb.build_system_matrix(geom)
    y, lam = golden["ell_y"], golden["ell_w"]
    prior = mb.PriorParams(kind, 20.0, 2.0, 1.2, 1.0, 0.01)
    prob = mb.ReconProblem(geom, mats, y, lam, prior)
    x = np.random.default_rng(7).random(ns * ns).astype(np.float32) * 0.03
    g, norms = mb.map_gradient(prob, x)
    want = _np_gradient(mats, y, lam, x.astype(np.float64), kind, 20.0, 2.0, 1.2, 1.0, 0.01, prior.eps_reg, ns)
    assert np.linalg.norm(g - want) <= 1e-5 * np.linalg.norm(want)
    assert norms[0] == pytest.approx(np.linalg.norm(want), rel=1e-5)


def test_gradient_vanishes_at_the_map(golden):
    ns, nv, nc = 32, 45, 47
    geom = mb.Geometry(ns, 4.0, nv, nc, 4.0)
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), golden["ell_y"], golden["ell_w"],
                           mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01))
    _, at0 = mb.map_gradient(prob, np.zeros(ns * ns, np.float32))
    _, at_map = mb.map_gradient(prob, golden["ell_central"].astype(np.float32))
    # float32 image of a float64 fixed point: only rounding of x is left
    assert at_map[0] < 1e-4 * at0[0]


def test_back_project_is_the_transpose_of_forward_project():
    ns, nv, nc = 32, 45, 47
    geom = mb.Geometry(ns, 4.0, nv, nc, 4.0)
    mats = mb.build_system_matrix(geom)
    rng = np.random.default_rng(11)
    s = rng.standard_normal((nv, nc))
    x = rng.standard_normal(ns * ns)
    bp = mb.back_project(mats, s)
    want = sum(O.view_csr(m).T @ s[k] for k, m in enumerate(mats))
    s32 = s.astype(np.float32).astype(np.float64)
    want32 = sum(O.view_csr(m).astype(np.float32).astype(np.float64).T @ s32[k] for k, m in enumerate(mats))
    assert np.linalg.norm(bp - want32) <= 1e-12 * np.linalg.norm(want32) * 10
    assert np.linalg.norm(bp - want) <= 1e-6 * np.linalg.norm(want)
    # adjointness <A x, s> = <x, A^T s> (the reference's own check, tests/test_geometry.py)
    lhs = float(np.sum(mb.forward_project(mats, x) * s))
    assert lhs == pytest.approx(float(x @ bp), rel=1e-5)
    with pytest.raises(ValueError):
        mb.back_project(mats, s[:, :-1])
