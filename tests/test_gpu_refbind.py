"""The reference's compiled plug point (`_sweep`, icd.py:67-139) bound to the B200 library
(paper_1911_09278_b200.refbind.sweep -> mace_sweep_f64): float64, raster order, so it must
match the oracle / the reference's golden vectors to ~1e-12 (only the in-warp summation
order of theta1 differs)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import small_problem

from paper_1911_09278_b200 import refbind

pytestmark = pytest.mark.gpu

CASES = ["pq", "pg", "pg2", "pq2", "pg3"]


def _agent(g, name):
    seed, ns, nv, nc, beta, sx, N, agent, sigma, is_qg = g[f"{name}_meta"]
    mats, y, w = small_problem(int(seed), int(ns), int(nv), int(nc))
    prior = O.Prior(kind="qggmrf" if is_qg else "quadratic-mrf", beta=float(beta), sigma_x=float(sx))
    views = O.partition_views(int(nv), int(N))[int(agent)]
    return O.Agent(mats, y, w, views, int(N), float(sigma), prior, int(ns), state=g[f"{name}_x0"])


def _args(ag, v, s0, s1):
    pr = ag.prior
    quad = pr.kind == "quadratic-mrf"
    return (ag.state, v, ag.e, ag.col_ptr, ag.row_idx, ag.a_val, ag.lam, ag.curv, ag.nbr_idx, ag.nbr_w,
            ag.beta_eff, pr.eps_reg if quad else 0.0, ag.inv_sigma2, quad, pr.p, pr.q, pr.T, pr.sigma_x,
            ag.clamp, s0, s1)


@pytest.mark.parametrize("name", CASES)
def test_bound_sweep_matches_reference_passes(golden, name):
    ag = _agent(golden, name)
    v = golden[f"{name}_v"]
    dsq = refbind.sweep(*_args(ag, v, 0, ag.n))
    assert dsq > 0
    assert np.allclose(ag.state, golden[f"{name}_z1"], rtol=0, atol=1e-12)
    assert np.allclose(ag.e, golden[f"{name}_e1"], rtol=0, atol=1e-12)
    for _ in range(4):
        refbind.sweep(*_args(ag, v, 0, ag.n))
    assert np.allclose(ag.state, golden[f"{name}_z5"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("name", CASES)
def test_bound_sweep_pixel_range_and_return_value(golden, name):
    a, b = _agent(golden, name), _agent(golden, name)
    v = golden[f"{name}_v"]
    s0, s1 = 3, min(11, a.n)
    d_gpu = refbind.sweep(*_args(a, v, s0, s1))
    d_cpu = b.run_range(v, s0, s1)
    assert d_gpu == pytest.approx(d_cpu, rel=1e-12)
    assert np.allclose(a.state, b.state, rtol=0, atol=1e-13)
    assert np.allclose(a.e, b.e, rtol=0, atol=1e-13)


def test_bound_sweep_rejects_non_float64_state(golden):
    ag = _agent(golden, "pq")
    args = list(_args(ag, golden["pq_v"], 0, ag.n))
    args[0] = ag.state.astype(np.float32)
    with pytest.raises(TypeError):
        refbind.sweep(*args)
