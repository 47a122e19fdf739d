"""PnP denoisers (mirrors /root/reference/pkg/src/macetomo/denoisers.py's interface).

``make_denoiser(spec, n_side)`` returns an image-to-image callable, as the
reference does; any such callable may also be passed to ``mace_pnp_solve``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["DenoiserSpec", "make_denoiser", "denoise"]


@dataclass(frozen=True)
class DenoiserSpec:
    """kind in {identity, quadratic-prox, boxcar} (denoisers.py:26-40)."""

    kind: str = "identity"
    lam: float = 1.0
    radius: int = 1

    def __post_init__(self):
        if self.kind not in ("identity", "quadratic-prox", "boxcar"):
            raise ValueError(f"unknown denoiser kind {self.kind!r}")
        if self.lam < 0:
            raise ValueError("lam must be >= 0")
        if self.radius < 1:
            raise ValueError("radius must be >= 1")


def _identity(v):
    return np.array(v, dtype=np.float64)


_DENSE_LIMIT = 4096  # pixels up to which the quadratic prox is a dense Cholesky solve (denoisers.py:23)


def _laplacian(n_side: int):
    """Weighted 8-neighbourhood graph Laplacian L = D - W (models.py:169-176: x^T L x =
    sum over pairs of w (x_s - x_r)^2), assembled from neighbor_table (each pair seen from both
    ends, so D is the row sum of W)."""
    import scipy.sparse as sp

    from .models import neighbor_table

    nbr, w = neighbor_table(n_side)
    n = n_side * n_side
    s = np.repeat(np.arange(n), nbr.shape[1])
    r, ww = nbr.ravel(), w.ravel()
    ok = r >= 0
    W = sp.csr_matrix((ww[ok], (s[ok], r[ok])), shape=(n, n))
    return (sp.diags(np.asarray(W.sum(axis=1)).ravel()) - W).tocsr()


class QuadraticProx:
    """H(v) = argmin_z lam/2 z^T L z + 1/2 ||z - v||^2, i.e. (I + lam L) z = v (denoisers.py:43-65):
    a dense Cholesky factor up to _DENSE_LIMIT pixels, conjugate gradients (rtol 1e-10) above.
    A host callable, applied once per PnP iteration as the reference applies it."""

    def __init__(self, lam: float, n_side: int):
        import scipy.linalg as sla
        import scipy.sparse as sp

        self.n = n_side * n_side
        self._op = (sp.identity(self.n, format="csr") + lam * _laplacian(n_side)).tocsr()
        self._cho = sla.cho_factor(self._op.toarray()) if self.n <= _DENSE_LIMIT else None

    def __call__(self, v):
        import scipy.linalg as sla
        import scipy.sparse.linalg as spla

        v = np.asarray(v, dtype=np.float64)
        if self._cho is not None:
            return sla.cho_solve(self._cho, v)
        z, info = spla.cg(self._op, v, rtol=1e-10, atol=0.0, maxiter=10 * self.n)
        if info != 0:
            raise RuntimeError(f"quadratic-prox CG failed to converge (info={info})")
        return z


class Boxcar:
    """Mean over the (2 radius + 1)^2 window, renormalised by the in-image count at the borders
    (denoisers.py:68-89), from a summed-area table."""

    def __init__(self, radius: int, n_side: int):
        self.radius, self.n_side = int(radius), int(n_side)

    def __call__(self, v):
        m, r = self.n_side, self.radius
        sat = np.zeros((m + 1, m + 1))
        sat[1:, 1:] = np.asarray(v, dtype=np.float64).reshape(m, m).cumsum(0).cumsum(1)
        i = np.arange(m)
        lo, hi = np.maximum(i - r, 0), np.minimum(i + r + 1, m)
        box = sat[np.ix_(hi, hi)] - sat[np.ix_(lo, hi)] - sat[np.ix_(hi, lo)] + sat[np.ix_(lo, lo)]
        return (box / np.outer(hi - lo, hi - lo)).ravel()


_BUILT = {}


def make_denoiser(spec: DenoiserSpec, n_side: int):
    """The reference's built-in denoisers (denoisers.py:92-106), cached per (spec, n_side)."""
    if spec.kind == "identity":
        return _identity
    key = (spec, int(n_side))
    if key not in _BUILT:
        if len(_BUILT) >= 32:
            _BUILT.clear()
        _BUILT[key] = QuadraticProx(spec.lam, n_side) if spec.kind == "quadratic-prox" else Boxcar(spec.radius, n_side)
    return _BUILT[key]


def denoise(spec: DenoiserSpec, v, n_side: int):
    return make_denoiser(spec, n_side)(v)


# --------------------------------------------------------------------------- K5: CNN denoiser agent

CNN_LAYERS, CNN_CHANNELS = 17, 64


def to_bf16_bits(a) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def from_bf16_bits(b) -> np.ndarray:
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def cnn_weights(seed: int = 0, scale: float = 0.1) -> list:
    """BASELINE config 3: 17 bias-free 3x3 conv layers (1->64, 15x 64->64, 64->1), He-normal
    from `seed` times `scale`, stored as bf16 (returned as float32 arrays holding bf16 values,
    PyTorch OIHW shapes)."""
    rng = np.random.default_rng(seed)
    shapes = [(CNN_CHANNELS, 1)] + [(CNN_CHANNELS, CNN_CHANNELS)] * 15 + [(1, CNN_CHANNELS)]
    out = []
    for oc, ic in shapes:
        std = np.sqrt(2.0 / (ic * 9)) * scale
        w = (rng.standard_normal((oc, ic, 3, 3)) * std).astype(np.float32)
        out.append(from_bf16_bits(to_bf16_bits(w)).reshape(oc, ic, 3, 3))
    return out


class CnnDenoiser:
    """H(v) = v - net(v) with the 17-layer CNN on the tensor cores (kernel K5).

    Usable as a plain callable (host round trip) or, inside ``mace_pnp_solve``, on the
    device: ``device_apply(plan)`` maps the consensus average to G_H without leaving HBM.
    """

    def __init__(self, n_side: int, weights=None, seed: int = 0, device: int = 0):
        self.n_side = n_side
        self.weights = cnn_weights(seed) if weights is None else [np.asarray(w, np.float32) for w in weights]
        if len(self.weights) != CNN_LAYERS:
            raise ValueError("the denoiser has 17 layers")
        self._bits = np.concatenate([to_bf16_bits(w).ravel() for w in self.weights])
        self.device = device
        self._ctx = None
        self._loaded = set()
        self.last_ms = None

    def _load(self, ctx):
        from . import _native as N

        key = id(ctx) if not hasattr(ctx, "h") else ctx.h.value
        if key not in self._loaded:
            ctx.call("mace_cnn_set_weights", N.ptr(self._bits), CNN_LAYERS, CNN_CHANNELS)
            self._loaded.add(key)

    def device_apply(self, plan):
        self._load(plan)
        plan.call("mace_cnn_apply")

    def layer(self, index: int, x_bits: np.ndarray) -> np.ndarray:
        """One 64 -> 64 layer alone on the tensor cores: middle layer `index` (0..14 = net layers
        2..16) of a (64, h, w) bf16 input given as uint16 bits; returns the bf16 bits of
        ReLU(conv) as (64, h, w).  Test hook for the per-layer rounding check."""
        from . import _native as N
        from .engine import _Context

        if self._ctx is None:
            self._ctx = _Context(self.device)
        self._load(self._ctx)
        x = np.ascontiguousarray(x_bits, np.uint16)
        if x.ndim != 3 or x.shape[0] != CNN_CHANNELS:
            raise ValueError("input must be (64, h, w) bf16 bits")
        out = np.empty_like(x)
        self._ctx.call("mace_cnn_layer", int(index), N.ptr(x), N.ptr(out), int(x.shape[1]), int(x.shape[2]))
        return out

    def __call__(self, v):
        import ctypes

        from . import _native as N
        from .engine import _Context

        if self._ctx is None:
            self._ctx = _Context(self.device)
        self._load(self._ctx)
        x = N.f32(np.asarray(v).reshape(-1))
        h = self.n_side
        w = x.shape[0] // h
        if h * w != x.shape[0]:
            raise ValueError("image size does not match n_side")
        out = np.empty_like(x)
        ms = ctypes.c_float(0.0)
        self._ctx.call("mace_cnn_run", N.ptr(x), N.ptr(out), int(h), int(w), ctypes.byref(ms))
        self.last_ms = ms.value
        return out.astype(np.float64)
