"""Converged float64 CPU-oracle MAP image for a config too large for oracle.Agent's scipy
stacking (config 2: 1.9e9 nnz; the Agent path would hold the per-view CSR, the stacked CSR
and the CSC at once, > 100 GB).  TEST INFRASTRUCTURE: writes tests/golden/central_c{C}.npz.

Same algorithm as oracle.icd_map_solve (icd.py:306-345): one agent with every view,
no proximal term, raster passes of oracle/sweep.c:orc_sweep (the _sweep restatement,
float64), e refreshed every 50 passes, stop when sqrt(sum alpha^2)/||z|| < tol.  Only
the construction is leaner:
  * the matrix comes from oracle.iter_system_matrix (the oracle tracer, one view at a time,
    in view order, in a process pool) and is checked against the reference's SHA-256
    (tests/golden/sysmat_digests.json, written by make_golden.py / make_c2_digest.py);
  * y and weights are synthesised exactly as gen.make_scan does (same phantom, same
    scipy per-view CSR product, same Poisson draw), so they are bit-identical to the
    arrays bench.py and the GPU tests use;
  * the stacked CSC (rows = view * n_ch + channel, ascending in each column, as
    icd.py:185-192's tocsc) is filled by a two-pass counting sort over the views.
The fixed point is unique (strictly convex MAP), so a warm start (--x0, e.g. the GPU image)
only shortens the run.  The stationarity |grad f(x)| / |grad f(0)| is evaluated in float64.

    python tools/cpu_central_lean.py --config 2 --x0 tests/golden/central_c2.npz --tol 1e-8
"""
import argparse
import hashlib
import importlib.util
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

# the workload recipe (phantom, Poisson draw, config table) without importing the package
_spec = importlib.util.spec_from_file_location("_gen", os.path.join(ROOT, "paper_1911_09278_b200", "gen.py"))
gen = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(gen)


def build(config, workers):
    c = gen.CONFIGS[config]
    ns, nv, nc = c["n_side"], c["n_views"], c["n_channels"]
    pitch = 1.0 if config == 0 else gen.pitch_for(ns)
    n = ns * ns
    phantom = gen.ellipse_phantom(ns, pitch, c["n_ellipses"], seed=0)
    t = time.time()
    h = hashlib.sha256()
    counts = np.zeros(n + 1, np.int64)
    proj = np.empty((nv, nc))
    for k, m in enumerate(O.iter_system_matrix(ns, pitch, nv, nc, pitch, workers)):
        h.update(m.row_ptr.astype(np.int64).tobytes())
        h.update(m.cols.astype(np.int32).tobytes())
        h.update(m.lens.astype(np.float64).tobytes())
        # gen.host_forward_project's exact expression
        proj[k] = sp.csr_matrix((m.lens, m.cols, m.row_ptr), shape=(m.n_channels, m.n_pixels)) @ phantom
        counts[1:] += np.bincount(m.cols, minlength=n)
    digest = h.hexdigest()
    print(f"pass 1 (trace, digest, projection): {time.time() - t:.1f} s; sha256 {digest}", flush=True)
    y, lam = gen.poisson_sinogram(proj, c["I0"], seed=1)
    col_ptr = np.cumsum(counts)
    nnz = int(col_ptr[-1])
    row_idx = np.empty(nnz, np.int64)
    a_val = np.empty(nnz, np.float64)
    fill = col_ptr[:-1].copy()
    t = time.time()
    for k, m in enumerate(O.iter_system_matrix(ns, pitch, nv, nc, pitch, workers)):
        rows = k * nc + np.repeat(np.arange(nc, dtype=np.int64), np.diff(m.row_ptr))
        order = np.argsort(m.cols, kind="stable")  # channel (= row) order kept inside a column
        cs = m.cols[order].astype(np.int64)
        start = np.r_[0, np.flatnonzero(np.diff(cs)) + 1]
        grp = np.repeat(start, np.diff(np.r_[start, cs.size]))
        pos = fill[cs] + (np.arange(cs.size) - grp)
        row_idx[pos] = rows[order]
        a_val[pos] = m.lens[order]
        u, cnt = cs[start], np.diff(np.r_[start, cs.size])
        fill[u] += cnt
    assert np.array_equal(fill, col_ptr[1:])
    print(f"pass 2 (CSC fill): {time.time() - t:.1f} s; nnz {nnz}", flush=True)
    return dict(ns=ns, n=n, y=y.ravel(), lam=lam.ravel(), col_ptr=col_ptr, row_idx=row_idx, a_val=a_val,
                digest=digest, phantom=phantom, beta=c["beta"])


def theta2(P, chunk=1 << 16):
    """sum_r a^2 lambda per column (icd.py:193-195)"""
    n, cp = P["n"], P["col_ptr"]
    out = np.empty(n)
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        a, b = cp[j0], cp[j1]
        v = P["a_val"][a:b] ** 2 * P["lam"][P["row_idx"][a:b]]
        out[j0:j1] = np.add.reduceat(v, cp[j0:j1] - a) if b > a else 0.0
        empty = cp[j0 + 1:j1 + 1] == cp[j0:j1]
        out[j0:j1][empty] = 0.0
    return out


def prior_grad(x, ns, beta, p=2.0, q=1.2, T=1.0, sx=0.01):
    """beta * d/dx sum_{pairs} w rho(x_s - x_r) (models.py:248-257), float64."""
    idx, w = O.neighbor_table(ns)
    g = np.zeros_like(x)
    for k in range(8):
        ok = idx[:, k] >= 0
        d = x[ok] - x[idx[ok, k]]
        g[ok] += w[ok, k] * O.qggmrf_influence(d, p, q, T, sx)
    return beta * g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-passes", type=int, default=3000)
    ap.add_argument("--x0", default="")
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--checkpoint", default="/tmp/central_lean_ckpt.npy")
    a = ap.parse_args()
    P = build(a.config, a.workers or None)
    digests = json.load(open(os.path.join(ROOT, "tests", "golden", "sysmat_digests.json")))
    ref_digest = digests.get(f"c{a.config}", {}).get("sha256")
    print("reference digest", ref_digest, "match" if ref_digest == P["digest"] else "MISMATCH / absent", flush=True)
    if ref_digest is not None and ref_digest != P["digest"]:
        raise SystemExit("oracle matrix differs from the reference's")
    n, ns = P["n"], P["ns"]
    A = sp.csc_matrix((P["a_val"], P["row_idx"], P["col_ptr"]), shape=(P["y"].size, n))
    curv = theta2(P)
    nbr_idx, nbr_w = O.neighbor_table(ns)
    beta = P["beta"]
    z = np.zeros(n)
    if a.x0:
        z = np.load(a.x0)["image"].astype(np.float64) if a.x0.endswith(".npz") else np.load(a.x0).astype(np.float64)
    x0 = z.copy()
    v = np.zeros(n)
    y, lam = P["y"], P["lam"]

    def residual(x):
        return y - A @ x

    e = residual(z)
    g0 = A.T @ (lam * y)  # |grad f(0)|: data part only (prior gradient vanishes at 0)
    g0n = float(np.linalg.norm(g0))
    L = O.lib()
    ptr = O._ptr
    hist = []
    t = time.time()
    passes = 0
    converged = False
    for k in range(a.max_passes):
        dsq = L.orc_sweep(ptr(z), ptr(v), ptr(e), ptr(P["col_ptr"]), ptr(P["row_idx"]), ptr(P["a_val"]), ptr(lam),
                          ptr(curv), ptr(nbr_idx), ptr(nbr_w), beta, 0.0, 0.0, 0, 2.0, 1.2, 1.0, 0.01, 0, 0, n)
        passes += 1
        if passes % O.REFRESH_EVERY == 0:
            e = residual(z)
            np.save(a.checkpoint, z)
        rel = float(np.sqrt(dsq) / max(np.linalg.norm(z), 1e-300))
        hist.append(rel)
        if passes % 5 == 0 or rel < a.tol:
            print(f"pass {passes}: relnorm {rel:.3e}  {time.time() - t:.0f} s", flush=True)
        if rel < a.tol:
            converged = True
            break
    e = residual(z)
    g = -(A.T @ (lam * e)) + prior_grad(z, ns, beta)
    ratio = float(np.linalg.norm(g)) / g0n
    start_gap = float(np.linalg.norm(z - x0) / np.linalg.norm(z))
    print(f"converged {converged} after {passes} passes, {time.time() - t:.0f} s; |grad f|/|grad f(0)| = "
          f"{ratio:.3e}; nrmse(x0, x*) = {start_gap:.3e}", flush=True)
    like = 0.5 * float(np.dot(lam * e, e))
    cost = like + O.prior_cost(z, "qggmrf", beta, 2.0, 1.2, 1.0, 0.01, 0.0, ns)
    out = a.out or os.path.join(ROOT, "tests", "golden", f"central_c{a.config}.npz")
    np.savez_compressed(out, image=z.astype(np.float32), passes=passes, converged=converged, cost=cost,
                        relnorm=np.array(hist), beta=beta, grad_ratio=ratio, tol=a.tol, sha256=P["digest"],
                        nrmse_x0=start_gap, nrmse_phantom=O.nrmse(z, P["phantom"]),
                        how="oracle icd_map_solve (float64 raster orc_sweep, tools/cpu_central_lean.py)"
                            + (f", warm start {os.path.basename(a.x0)}" if a.x0 else ""))
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main()
