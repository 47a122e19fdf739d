"""Multi-slice batches (BASELINE config 4 recipe): slices share one operator and run as
concurrent agents on the same super-voxel tiles.  Each slice must reach its own MAP fixed
point (the CPU oracle's converged icd_map_solve of that slice)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen

pytestmark = pytest.mark.gpu


def test_batch_slices_reach_their_own_map():
    ns, nv, nc, S, N = 32, 45, 47, 5, 4
    pitch = 128.0 / ns
    geom = mb.Geometry(ns, pitch, nv, nc, pitch)
    mats = mb.build_system_matrix(geom)
    prior = mb.PriorParams("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01)
    probs, refs = [], []
    for s in range(S):
        ph = gen.ellipse_phantom(ns, pitch, 10, seed=100 + s)
        y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 1e4, seed=200 + s)
        probs.append(mb.ReconProblem(geom, mats, y, lam, prior))
        x, _ = O.icd_map_solve(mats, y, lam, O.Prior("qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01), ns, tol=1e-10,
                               max_passes=5000)
        refs.append(x)
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=2.5e-4, max_outer=3000, tol=1e-300, residuals="none",
                        sv_side=4)
    try:
        res = mb.mace_solve_batch(probs, cfg)
    except mb.ConvergenceError as err:
        res = err.last_iterate
    assert len(res) == S
    for s in range(S):
        assert res[s].stack.shape == (N, ns * ns)
        assert O.nrmse(res[s].image, refs[s]) < 1e-3, (s, O.nrmse(res[s].image, refs[s]))


def test_batch_rejects_mismatched_slices():
    geom = mb.Geometry(8, 1.0, 8, 9, 1.0)
    mats = mb.build_system_matrix(geom)
    other = mb.build_system_matrix(geom)
    z = np.zeros((8, 9))
    p1 = mb.ReconProblem(geom, mats, z, z + 1, mb.PriorParams())
    p2 = mb.ReconProblem(geom, other, z, z + 1, mb.PriorParams())
    with pytest.raises(ValueError):
        mb.mace_solve_batch([p1, p2], mb.MaceConfig(n_subsets=2, residuals="none"))
