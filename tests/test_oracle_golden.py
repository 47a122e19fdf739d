"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference itself.

Fixtures: tests/golden/golden_small.npz (tests/golden/make_golden.py).  These
run without a GPU and gate every parity claim made against the oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import small_problem, unpack_views
from golden.make_golden import GEOMS


@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_tracer_bit_exact_vs_reference(golden, gi):
    ns, pp, nv, nc, cp = GEOMS[gi]
    mats = O.build_system_matrix(ns, pp, nv, nc, cp)
    ref = unpack_views(golden, f"geom{gi}", nv, nc, ns * ns)
    for m, r in zip(mats, ref):
        assert np.array_equal(m.row_ptr, r.row_ptr)
        assert np.array_equal(m.cols, r.cols)
        assert np.array_equal(m.lens, r.lens)  # bitwise float64


@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_forward_project_vs_reference(golden, gi):
    ns, pp, nv, nc, cp = GEOMS[gi]
    ref = unpack_views(golden, f"geom{gi}", nv, nc, ns * ns)
    fp = O.forward_project(ref, golden[f"geom{gi}_x"])
    assert np.allclose(fp, golden[f"geom{gi}_fp"], rtol=0, atol=1e-12)


def test_partitions_vs_reference(golden):
    for nv, N, i, count, total in golden["partitions"]:
        sub = O.partition_views(int(nv), int(N))[int(i)]
        assert len(sub) == count and sum(sub) == total
    with pytest.raises(ValueError):
        O.partition_views(3, 4)


@pytest.mark.parametrize("params", [(2.0, 1.2, 1.0, 0.01), (2.0, 1.2, 1.0, 0.5), (1.5, 1.1, 2.0, 0.3),
                                    (2.0, 2.0, 1.0, 1.0)])
def test_potential_functions_vs_reference(golden, params):
    p, q, T, sx = params
    key = f"qg_{p}_{q}_{T}_{sx}"
    d = golden[key + "_d"]
    L = O.lib()
    infl = np.array([L.orc_influence(x, p, q, T, sx) for x in d])
    coef = np.array([L.orc_coef(x, p, q, T, sx) for x in d])
    assert np.allclose(infl, golden[key + "_infl"], rtol=1e-13, atol=0)
    assert np.allclose(coef, golden[key + "_coef"], rtol=1e-13, atol=0)
    assert np.allclose(O.qggmrf_potential(d, p, q, T, sx), golden[key + "_pot"], rtol=1e-13, atol=0)
    assert np.allclose(O.qggmrf_influence(d, p, q, T, sx), golden[key + "_infl"], rtol=1e-13, atol=0)


CASES = ["pq", "pg", "pg2", "pq2", "pg3"]


def _agent_from_golden(g, name):
    seed, ns, nv, nc, beta, sx, N, agent, sigma, is_qg = g[f"{name}_meta"]
    ns, nv, nc, N, agent = int(ns), int(nv), int(nc), int(N), int(agent)
    mats, y, w = small_problem(int(seed), ns, nv, nc)
    assert np.array_equal(y, g[f"{name}_y"]) and np.array_equal(w, g[f"{name}_w"])
    prior = O.Prior(kind="qggmrf" if is_qg else "quadratic-mrf", beta=float(beta), sigma_x=float(sx))
    views = O.partition_views(nv, N)[agent]
    ag = O.Agent(mats, y, w, views, N, float(sigma), prior, ns, state=g[f"{name}_x0"])
    return ag


@pytest.mark.parametrize("name", CASES)
def test_agent_layout_bit_exact(golden, name):
    ag = _agent_from_golden(golden, name)
    assert np.array_equal(ag.col_ptr, golden[f"{name}_colptr"])
    assert np.array_equal(ag.row_idx, golden[f"{name}_rowidx"])
    assert np.array_equal(ag.a_val, golden[f"{name}_aval"])
    assert np.allclose(ag.curv, golden[f"{name}_curv"], rtol=1e-14, atol=0)
    assert np.allclose(ag.e, golden[f"{name}_e0"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", CASES)
def test_partial_update_vs_reference(golden, name):
    ag = _agent_from_golden(golden, name)
    v = golden[f"{name}_v"]
    z1 = ag.partial_update(v)
    assert np.allclose(z1, golden[f"{name}_z1"], rtol=0, atol=1e-12)
    assert np.allclose(ag.e, golden[f"{name}_e1"], rtol=0, atol=1e-12)
    for _ in range(4):
        z5 = ag.partial_update(v)
    assert np.allclose(z5, golden[f"{name}_z5"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("name", CASES)
def test_pixel_update_vs_reference(golden, name):
    ag = _agent_from_golden(golden, name)
    s = min(7, ag.n - 1)
    before = ag.state[s]
    ag.run_range(golden[f"{name}_v"], s, s + 1)
    assert ag.state[s] - before == pytest.approx(golden[f"{name}_alpha7"][0], rel=1e-12, abs=1e-15)


def _mq_agents(golden, sigma=0.2, pnp=False):
    mats, y, w = small_problem(31, 8, 16, 11)
    assert np.array_equal(y, golden["mq_y"])
    prior = O.Prior(kind="qggmrf", beta=1.0, sigma_x=0.5)
    return mats, y, w, prior, O.build_agents(mats, y, w, 4, sigma, prior, 8, pnp=pnp)


def test_mace_fixed_budget_vs_reference(golden):
    _, _, _, _, agents = _mq_agents(golden)
    run = O.mace_run(agents, 12, 0.8)
    assert np.allclose(run.stack, golden["mq_stack"], rtol=0, atol=1e-11)
    assert np.allclose(run.image, golden["mq_image"], rtol=0, atol=1e-11)
    assert np.allclose(run.relnorms, golden["mq_relnorm"], rtol=1e-9)


def test_mace_deterministic_across_workers(golden):
    _, _, _, _, a1 = _mq_agents(golden)
    _, _, _, _, a4 = _mq_agents(golden)
    r1 = O.mace_run(a1, 12, 0.8, workers=None)
    r4 = O.mace_run(a4, 12, 0.8, workers=4)
    assert np.array_equal(r1.image, r4.image)


def test_centralized_icd_vs_reference(golden):
    mats, y, w, prior, _ = _mq_agents(golden)
    x, _ = O.icd_map_solve(mats, y, w, prior, 8, tol=1e-12, max_passes=4000)
    assert O.nrmse(x, golden["mq_central"]) < 1e-10
    # MACE fixed point == centralized MAP (reference tests/test_mace.py:184-192)
    assert O.nrmse(golden["mq_converged"], golden["mq_central"]) < 1e-5


def _boxcar(n_side):
    """Restates the reference's boxcar denoiser (denoisers.py:67-96) for the PnP fixture."""
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


def test_mace_pnp_fixed_budget_vs_reference(golden):
    mats, y, w, prior, _ = _mq_agents(golden)
    agents = O.build_agents(mats, y, w, 4, 0.1, prior, 8, pnp=True)
    run = O.mace_run(agents, 10, 0.8, denoiser=_boxcar(8))
    assert np.allclose(run.stack, golden["mp_stack"], rtol=0, atol=1e-11)
    assert np.allclose(run.image, golden["mp_image"], rtol=0, atol=1e-11)


def test_ellipse_problem_and_costs_vs_reference(golden):
    from paper_1911_09278_b200 import gen

    phantom = gen.ellipse_phantom(32, 4.0, n_ellipses=10, seed=3)
    assert np.array_equal(phantom, golden["ell_phantom"])
    mats = O.build_system_matrix(32, 4.0, 45, 47, 4.0)
    y, lam = gen.poisson_sinogram(O.forward_project(mats, phantom), 1e4, seed=4)
    assert np.array_equal(y, golden["ell_y"]) and np.array_equal(lam, golden["ell_w"])
    x = golden["ell_central"]
    cost = O.likelihood_cost(mats, y, lam, x) + O.prior_cost(x, "qggmrf", 20.0, 2.0, 1.2, 1.0, 0.01, 0, 32)
    assert cost == pytest.approx(golden["ell_cost_central"][0], rel=1e-12)


def _digest(mats):
    import hashlib

    h = hashlib.sha256()
    for m in mats:
        h.update(np.ascontiguousarray(m.row_ptr, np.int64).tobytes())
        h.update(np.ascontiguousarray(m.cols, np.int32).tobytes())
        h.update(np.ascontiguousarray(m.lens, np.float64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name,workers", [("c0", 1), ("c0", 4), ("c1", 8)])
def test_parallel_oracle_tracer_matches_reference_digest(name, workers):
    """oracle.iter_system_matrix (views traced by a process pool, consumed in view order; the
    path bench.py's reference arm and tools/cpu_central_lean.py use) reproduces the reference's
    full system matrix: SHA-256 written by the reference itself (sysmat_digests.json; config 2's
    digest is checked by cpu_central_lean.py when it builds the config-2 oracle MAP)."""
    import json
    import os

    from conftest import GOLDEN

    d = json.load(open(os.path.join(GOLDEN, "sysmat_digests.json")))
    assert "c2" in d and d["c2"]["nnz"] == 1922520128
    ns, pp, nv, nc, cp = d[name]["params"]
    mats = list(O.iter_system_matrix(int(ns), pp, int(nv), int(nc), cp, workers=workers))
    assert _digest(mats) == d[name]["sha256"]


def test_reference_arm_scan_equals_gpu_arm_scan():
    """bench.reference_scan (oracle tracer + gen recipe, no CUDA library) yields bit-identical y and
    weights to gen.make_scan (the GPU arm's), so both arms solve the same problem."""
    import bench

    from paper_1911_09278_b200 import gen

    _, _, mats_r, y_r, lam_r = bench.reference_scan(0, workers=4)
    _, mats_g, _, y_g, lam_g = gen.make_scan(0)
    assert np.array_equal(y_r, y_g) and np.array_equal(lam_r, lam_g)
    assert all(np.array_equal(a.cols, b.cols) and np.array_equal(a.lens, b.lens) for a, b in zip(mats_r, mats_g))
