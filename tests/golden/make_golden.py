"""Generate the golden vectors in tests/golden/ by running the REFERENCE package.

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --hashes   # + c0/c1 system-matrix digests (~1 min)

The reference is copied to /tmp/refpkg first because numba writes its cache
beside the sources and /root/reference is read-only.  Every fixture stores its
own inputs, so the tests never need the reference at run time.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
REF_COPY = "/tmp/refpkg"


def import_reference():
    if not os.path.isdir(REF_COPY):
        shutil.copytree(REF_SRC, REF_COPY)
    sys.path.insert(0, os.path.join(REF_COPY, "src"))
    import macetomo  # noqa: F401

    return macetomo


def mat_digest(matrices) -> str:
    """SHA-256 over (row_ptr int64, cols int32, lens float64) of every view, in order."""
    h = hashlib.sha256()
    for m in matrices:
        h.update(np.ascontiguousarray(m.row_ptr, np.int64).tobytes())
        h.update(np.ascontiguousarray(m.cols, np.int32).tobytes())
        h.update(np.ascontiguousarray(m.lens, np.float64).tobytes())
    return h.hexdigest()


def pack_matrices(matrices):
    return {
        "row_ptr": np.concatenate([m.row_ptr for m in matrices]).astype(np.int64),
        "cols": np.concatenate([m.cols for m in matrices]).astype(np.int32),
        "lens": np.concatenate([m.lens for m in matrices]).astype(np.float64),
        "nnz_per_view": np.array([m.nnz for m in matrices], np.int64),
    }


GEOMS = [
    # n_side, pixel_pitch, n_views, n_channels, channel_pitch
    (1, 1.0, 1, 1, 1.0),
    (4, 1.0, 2, 3, 1.0),
    (5, 1.0, 8, 7, 5 / 7 * 1.1),
    (6, 1.0, 12, 9, 6 / 9 * 1.1),
    (8, 1.0, 12, 11, 8 / 11 * 1.1),
    (16, 0.5, 30, 25, 0.5),
    (32, 1.0, 45, 47, 1.0),
    (32, 4.0, 64, 47, 4.0),
    (13, 0.37, 17, 23, 0.29),
]


def small_problem(mt, seed, n_side, n_views, n_channels, kind, beta, sigma_x):
    """Same recipe as the reference's tests/conftest.py:17-32 (random y, weights in [0.5, 1.5))."""
    rng = np.random.default_rng(seed)
    geom = mt.Geometry(n_side=n_side, pixel_pitch=1.0, n_views=n_views, n_channels=n_channels,
                       channel_pitch=n_side / n_channels * 1.1)
    mats = mt.build_system_matrix(geom)
    y = rng.standard_normal((n_views, n_channels))
    w = 0.5 + rng.random((n_views, n_channels))
    prior = mt.PriorParams(kind=kind, beta=beta, sigma_x=sigma_x)
    return mt.ReconProblem(geom, mats, y, w, prior)


def ellipse_problem(mt, n_side, n_views, n_channels, seed, beta, I0=1e4):
    """Counts-weighted ellipse problem (the bench recipe, in miniature), fed to the reference."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1911_09278_b200 import gen

    pitch = 128.0 / n_side
    geom = mt.Geometry(n_side=n_side, pixel_pitch=pitch, n_views=n_views, n_channels=n_channels,
                       channel_pitch=pitch)
    mats = mt.build_system_matrix(geom)
    phantom = gen.ellipse_phantom(n_side, pitch, n_ellipses=10, seed=seed)
    proj = mt.forward_project(mats, phantom)
    y, lam = gen.poisson_sinogram(proj, I0, seed=seed + 1)
    prior = mt.PriorParams(kind="qggmrf", beta=beta, p=2.0, q=1.2, T=1.0, sigma_x=0.01)
    return mt.ReconProblem(geom, mats, y, lam, prior), phantom


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hashes", action="store_true")
    args = ap.parse_args()
    mt = import_reference()
    from macetomo import icd as ricd
    from macetomo import mace as rmace

    out = {}

    # --- geometry: full system matrices at small sizes (geometry.py:228-258)
    for gi, (ns, pp, nv, nc, cp) in enumerate(GEOMS):
        geom = mt.Geometry(ns, pp, nv, nc, cp)
        mats = mt.build_system_matrix(geom)
        for k, v in pack_matrices(mats).items():
            out[f"geom{gi}_{k}"] = v
        out[f"geom{gi}_params"] = np.array([ns, pp, nv, nc, cp], np.float64)
        x = np.random.default_rng(gi).standard_normal(ns * ns)
        out[f"geom{gi}_x"] = x
        out[f"geom{gi}_fp"] = mt.forward_project(mats, x)

    # --- partitions (geometry.py:161-174)
    parts = []
    for nv, N in [(8, 2), (8, 1), (7, 3), (180, 4), (720, 8), (1440, 16), (13, 13)]:
        for s in mt.partition_views(nv, N):
            parts.append([nv, N, s.subset_index, len(s.view_indices), sum(s.view_indices)])
    out["partitions"] = np.array(parts, np.int64)

    # --- potential functions (icd.py:45-64 / models.py:121-166)
    d = np.concatenate([-np.logspace(-12, 1, 40), [0.0], np.logspace(-12, 1, 40)])
    for (p, q, T, sx) in [(2.0, 1.2, 1.0, 0.01), (2.0, 1.2, 1.0, 0.5), (1.5, 1.1, 2.0, 0.3), (2.0, 2.0, 1.0, 1.0)]:
        key = f"qg_{p}_{q}_{T}_{sx}"
        out[key + "_d"] = d
        out[key + "_infl"] = np.array([ricd._qg_influence(x, p, q, T, sx) for x in d])
        out[key + "_coef"] = np.array([ricd._qg_coef(x, p, q, T, sx) for x in d])
        out[key + "_pot"] = mt.models.qggmrf_potential(d, p, q, T, sx)

    # --- one-pass and multi-pass partial updates (icd.py:175-283)
    cases = [
        ("pq", 21, 6, 12, 9, "quadratic-mrf", 1.5, 1.0, 3, 1, 0.6),
        ("pg", 21, 6, 12, 9, "qggmrf", 1.5, 0.8, 3, 1, 0.6),
        ("pg2", 5, 8, 12, 11, "qggmrf", 0.8, 0.3, 4, 2, 0.4),
        ("pq2", 31, 8, 12, 11, "quadratic-mrf", 0.8, 1.0, 2, 0, 0.4),
        ("pg3", 7, 13, 20, 17, "qggmrf", 2.0, 0.05, 5, 4, 0.3),
    ]
    for name, seed, ns, nv, nc, kind, beta, sx, N, agent, sigma in cases:
        prob = small_problem(mt, seed, ns, nv, nc, kind, beta, sx)
        subsets = mt.partition_views(nv, N)
        rng = np.random.default_rng(seed + 1000)
        x0 = rng.standard_normal(prob.n)
        v = rng.standard_normal(prob.n)
        ws = mt.AgentWorkspace(prob, subsets[agent], N, sigma=sigma, state=x0)
        out[f"{name}_meta"] = np.array([seed, ns, nv, nc, beta, sx, N, agent, sigma, kind == "qggmrf"])
        out[f"{name}_y"] = prob.y
        out[f"{name}_w"] = prob.weights
        out[f"{name}_x0"] = x0
        out[f"{name}_v"] = v
        out[f"{name}_colptr"] = ws.col_ptr
        out[f"{name}_rowidx"] = ws.row_idx
        out[f"{name}_aval"] = ws.a_val
        out[f"{name}_curv"] = ws.curv_data
        out[f"{name}_e0"] = ws.error_sinogram.copy()
        z1 = mt.partial_update_prox(ws, v)
        out[f"{name}_z1"] = z1
        out[f"{name}_e1"] = ws.error_sinogram.copy()
        for _ in range(4):
            z5 = mt.partial_update_prox(ws, v)
        out[f"{name}_z5"] = z5
        # single-pixel update KAT (icd.py:256-269)
        ws2 = mt.AgentWorkspace(prob, subsets[agent], N, sigma=sigma, state=x0)
        out[f"{name}_alpha7"] = np.array([mt.pixel_update(ws2, min(7, prob.n - 1), v)])

    # --- MACE runs at a fixed budget (mace.py:276-365), conventional + PnP
    def run_fixed(fn, prob, cfg, **kw):
        try:
            res = fn(prob, cfg, **kw)
        except ricd.ConvergenceError as err:
            res = err.last_iterate
        return res

    prob = small_problem(mt, 31, 8, 16, 11, "qggmrf", 1.0, 0.5)
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=12, tol=1e-300, residuals="none")
    res = run_fixed(mt.mace_solve, prob, cfg)
    out["mq_y"], out["mq_w"] = prob.y, prob.weights
    out["mq_image"], out["mq_stack"] = res.image, res.stack
    out["mq_relnorm"] = np.array([r["relnorm"] for r in res.log.rows])
    x_central = mt.icd_map_solve(prob, tol=1e-12, max_passes=4000)
    out["mq_central"] = x_central
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, tol=1e-10, max_outer=12000, residuals="none")
    out["mq_converged"] = mt.mace_solve(prob, cfg).image

    # PnP with a custom callable (mace.py:385-404) — boxcar radius 1
    H = mt.make_denoiser(mt.DenoiserSpec(kind="boxcar", radius=1), prob.geom.n_side)
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=0.1, mode="pnp",
                           denoiser=mt.DenoiserSpec(kind="identity"), max_outer=10, tol=1e-300,
                           residuals="none")
    res = run_fixed(mt.mace_pnp_solve, prob, cfg, denoiser=H)
    out["mp_image"], out["mp_stack"] = res.image, res.stack
    out["mp_relnorm"] = np.array([r["relnorm"] for r in res.log.rows])

    # counts-weighted ellipse problem, miniature of config 0 (N=4, rho=0.8, qggmrf p=2 q=1.2)
    eprob, phantom = ellipse_problem(mt, 32, 45, 47, seed=3, beta=20.0)
    out["ell_phantom"], out["ell_y"], out["ell_w"] = phantom, eprob.y, eprob.weights
    cfg = rmace.MaceConfig(n_subsets=4, rho=0.8, sigma=3e-4, max_outer=30, tol=1e-300, residuals="none")
    res = run_fixed(mt.mace_solve, eprob, cfg)
    out["ell_image30"], out["ell_stack30"] = res.image, res.stack
    out["ell_relnorm"] = np.array([r["relnorm"] for r in res.log.rows])
    out["ell_central"] = mt.icd_map_solve(eprob, tol=1e-11, max_passes=5000)
    out["ell_cost_central"] = np.array([mt.map_cost(eprob, out["ell_central"])])

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("wrote golden_small.npz", os.path.getsize(os.path.join(HERE, "golden_small.npz")), "bytes")

    if args.hashes:
        digests = {}
        for name, (ns, pp, nv, nc, cp) in {
            "c0": (128, 1.0, 180, 185, 1.0),
            "c1": (512, 0.25, 720, 725, 0.25),
        }.items():
            mats = mt.build_system_matrix(mt.Geometry(ns, pp, nv, nc, cp))
            digests[name] = {"params": [ns, pp, nv, nc, cp], "sha256": mat_digest(mats),
                             "nnz": int(sum(m.nnz for m in mats))}
            print(name, digests[name])
        with open(os.path.join(HERE, "sysmat_digests.json"), "w") as fh:
            json.dump(digests, fh, indent=1)


if __name__ == "__main__":
    main()
