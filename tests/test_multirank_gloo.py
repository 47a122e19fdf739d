"""Multi-rank MACE host logic (agents sharded over ranks, one all-reduce of the stack sum +
norm scalars per iteration) on CPU with torch.distributed/gloo, world size 2 (and 3), using
the oracle-backed CPU plan (tests/cpu_backend.py) in place of the device plan."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import paper_1911_09278_b200 as mb
    from conftest import small_problem

    _, y, w = small_problem(31, 8, 16, 11)
    geom = mb.Geometry(8, 1.0, 16, 11, 8 / 11 * 1.1)
    return mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 1.0, sigma_x=0.5))


def _solve(comm, iters, pnp=False, tol=1e-300):
    import paper_1911_09278_b200 as mb
    from cpu_backend import CpuPlan

    prob = _problem()
    if pnp:
        cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.1, mode="pnp", denoiser=mb.DenoiserSpec("identity"),
                            max_outer=iters, tol=tol, residuals="none")
        H = lambda v: 0.5 * np.asarray(v) + 0.5 * np.mean(v)  # noqa: E731 - any callable
        fn = lambda: mb.mace_pnp_solve(prob, cfg, comm=comm, denoiser=H, _backend=CpuPlan)  # noqa: E731
    else:
        cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=iters, tol=tol, residuals="none")
        fn = lambda: mb.mace_solve(prob, cfg, comm=comm, _backend=CpuPlan)  # noqa: E731
    try:
        res = fn()
    except mb.ConvergenceError as err:
        res = err.last_iterate
    return res.image, res.stack, [r["relnorm"] for r in res.log.rows], res.converged


def _worker(rank, world, port, q, iters, pnp, tol):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = _solve(True, iters, pnp, tol)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run_world(world, iters, pnp=False, tol=1e-300):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, iters, pnp, tol)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_matches_single_rank_and_reference(world, golden):
    iters = 12
    single = _solve(None, iters)
    multi = _run_world(world, iters)
    for r in range(world):  # every rank holds the same consensus image and the gathered stack
        img, stack, rel, _ = multi[r]
        assert np.allclose(img, single[0], rtol=0, atol=1e-12)
        assert np.allclose(stack, single[1], rtol=0, atol=1e-12)
        assert np.allclose(rel, single[2], rtol=1e-10)
    # and the single-rank CPU plan reproduces the reference's own 12-iteration run
    assert np.allclose(single[1], golden["mq_stack"], rtol=0, atol=1e-11)
    assert np.allclose(single[0], golden["mq_image"], rtol=0, atol=1e-11)


def test_multirank_stop_test_is_global():
    single = _solve(None, 5000, tol=1e-6)
    multi = _run_world(2, 5000, tol=1e-6)
    assert single[3] and multi[0][3] and multi[1][3]
    assert len(multi[0][2]) == len(single[2]) == len(multi[1][2])


def test_multirank_pnp_callable():
    single = _solve(None, 8, pnp=True)
    multi = _run_world(2, 8, pnp=True)
    assert np.allclose(multi[0][0], single[0], rtol=0, atol=1e-12)
    assert np.allclose(multi[1][1], single[1], rtol=0, atol=1e-12)
