"""Seeded synthetic workload for the benchmark configurations (BASELINE.json:configs).

The reference ships only fixed phantoms and a Gaussian noise model
(/root/reference/pkg/src/macetomo/sim.py:58-120); BASELINE asks for seeded
random ellipses and Poisson counts, so this module defines that recipe.  The
same arrays feed the CPU oracle and the GPU path (decisions recorded in
DESIGN.md §3):

* field of view fixed at 128 mm; pixel pitch = channel pitch = 128 / n_side mm;
* phantom = 0.02 mm^-1 disk (radius 0.9 x half-FOV) + K ellipses with values
  U[0.005, 0.05] mm^-1 painted in draw order, 2x2 supersampled;
* counts ~ Poisson(I0 exp(-A x)) clamped >= 1; y = -log(counts / I0); lambda = counts.
"""

from __future__ import annotations

import numpy as np

FOV_MM = 128.0

# BASELINE.json:configs -> (n_side, n_views, n_channels, n_agents, iterations, I0, n_ellipses, slices)
# beta is the reference-convention qGGMRF strength (p=2, q=1.2, T=1, sigma_x=0.01); sigma is the
# agents' proximal parameter.  BASELINE leaves both open; values and probes in DESIGN.md §3
# (config 2: sigma 7e-4 reaches NRMSE 1e-3 in 5,561 iterations, 3.5e-4 needs 22,126, 1e-3 diverges;
# the same at the 8-GPU per-agent staleness, tools/probe_sigma.py, profiles/r02_probe_c2_sigma.log).
CONFIGS = {
    0: dict(n_side=128, n_views=180, n_channels=185, n_agents=4, iters=30, I0=1e4, n_ellipses=10, slices=1,
            beta=100.0, sigma=2.5e-4),
    1: dict(n_side=512, n_views=720, n_channels=725, n_agents=8, iters=40, I0=1e4, n_ellipses=10, slices=1,
            beta=25.0, sigma=3.5e-4),
    2: dict(n_side=1024, n_views=1440, n_channels=1450, n_agents=16, iters=50, I0=5e3, n_ellipses=40, slices=1,
            beta=4.0, sigma=7e-4),
    # PnP agents run at sqrt(N) sigma (mace.py:263-265): sigma = 3.5e-4 / sqrt(8) keeps them at c1's margin
    3: dict(n_side=512, n_views=720, n_channels=725, n_agents=8, iters=40, I0=1e4, n_ellipses=10, slices=1,
            beta=25.0, sigma=1.24e-4),
    4: dict(n_side=512, n_views=720, n_channels=725, n_agents=8, iters=30, I0=1e4, n_ellipses=10, slices=64,
            beta=25.0, sigma=3.5e-4),
}


def pitch_for(n_side: int, config: int | None = None) -> float:
    """Pixel = channel pitch.  Config 0 is 1 mm by BASELINE; the rest keep the 128 mm FOV."""
    return FOV_MM / n_side


def ellipse_phantom(n_side: int, pitch: float, n_ellipses: int = 10, seed: int = 0,
                    disk_value: float = 0.02, value_range=(0.005, 0.05)) -> np.ndarray:
    """Flat (n_side*n_side,) float64 attenuation image in mm^-1, row 0 at the top."""
    rng = np.random.default_rng(seed)
    half = 0.5 * n_side * pitch
    R = 0.9 * half
    # 2x2 supersampled pixel sample points
    sub = (np.arange(2 * n_side) + 0.5) * (pitch / 2.0)
    xs = sub - half
    ys = half - sub
    X, Y = np.meshgrid(xs, ys)
    img = np.where(X * X + Y * Y <= R * R, disk_value, 0.0)
    for _ in range(n_ellipses):
        r = 0.6 * R * np.sqrt(rng.random())
        phi = 2.0 * np.pi * rng.random()
        cx, cy = r * np.cos(phi), r * np.sin(phi)
        a = R * rng.uniform(0.05, 0.25)
        b = R * rng.uniform(0.05, 0.25)
        ang = np.pi * rng.random()
        val = rng.uniform(*value_range)
        c, s = np.cos(ang), np.sin(ang)
        dx, dy = X - cx, Y - cy
        u = (c * dx + s * dy) / a
        v = (-s * dx + c * dy) / b
        img = np.where(u * u + v * v <= 1.0, val, img)
    img = img.reshape(n_side, 2, n_side, 2).mean(axis=(1, 3))
    return np.ascontiguousarray(img.ravel())


def host_forward_project(matrices, x) -> np.ndarray:
    """Float64 host projection used only to synthesise data (identical for every arm)."""
    import scipy.sparse as sp

    x = np.asarray(x, np.float64)
    out = np.empty((len(matrices), matrices[0].n_channels))
    for k, m in enumerate(matrices):
        A = sp.csr_matrix((m.lens, m.cols, m.row_ptr), shape=(m.n_channels, m.n_pixels))
        out[k] = A @ x
    return out


def make_scan(config: int = 1, seed: int = 0, slice_index: int = 0, matrices=None):
    """(geometry, matrices, phantom, y, weights) for BASELINE config `config` (seeded)."""
    from .geometry import Geometry, build_system_matrix

    c = CONFIGS[config]
    ns = c["n_side"]
    pitch = 1.0 if config == 0 else pitch_for(ns)
    geom = Geometry(ns, pitch, c["n_views"], c["n_channels"], pitch)
    if matrices is None:
        matrices = build_system_matrix(geom)
    s = seed + 1000 * slice_index
    phantom = ellipse_phantom(ns, pitch, c["n_ellipses"], seed=s)
    y, lam = poisson_sinogram(host_forward_project(matrices, phantom), c["I0"], seed=s + 1)
    return geom, matrices, phantom, y, lam


def make_batch(config: int = 4, seed: int = 0, n_slices: int | None = None, device_fp: bool = True):
    """Config-4 batch: one geometry, `n_slices` seeded phantoms (seed + 1000 s), Poisson data.
    device_fp: project the phantoms with the GPU operator (K3, float32) instead of the float64
    host projector — 64 host projections at 512^2 take ~45 s; the data is synthetic either way."""
    from .geometry import Geometry, build_system_matrix

    c = CONFIGS[config]
    ns = c["n_side"]
    S = c["slices"] if n_slices is None else n_slices
    pitch = pitch_for(ns)
    geom = Geometry(ns, pitch, c["n_views"], c["n_channels"], pitch)
    mats = build_system_matrix(geom)
    if device_fp:
        from .engine import operator_for

        op = operator_for(mats)
        fp = lambda x: op.forward_project(x).astype(np.float64)  # noqa: E731
    else:
        fp = lambda x: host_forward_project(mats, x)  # noqa: E731
    phantoms, ys, lams = [], [], []
    for s in range(S):
        ph = ellipse_phantom(ns, pitch, c["n_ellipses"], seed=seed + 1000 * s)
        y, lam = poisson_sinogram(fp(ph), c["I0"], seed=seed + 1000 * s + 1)
        phantoms.append(ph)
        ys.append(y)
        lams.append(lam)
    return geom, mats, phantoms, ys, lams


def poisson_sinogram(proj: np.ndarray, I0: float, seed: int = 1):
    """counts ~ Poisson(I0 exp(-proj)), clamped >= 1; returns (y, weights=counts)."""
    rng = np.random.default_rng(seed)
    counts = rng.poisson(I0 * np.exp(-np.asarray(proj, np.float64))).astype(np.float64)
    np.maximum(counts, 1.0, out=counts)
    y = -np.log(counts / I0)
    return y, counts
