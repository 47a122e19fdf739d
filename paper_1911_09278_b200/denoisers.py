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


def make_denoiser(spec: DenoiserSpec, n_side: int):
    if spec.kind == "identity":
        return _identity
    raise NotImplementedError(
        f"built-in denoiser {spec.kind!r} is outside the B200 hot path; pass it as a callable "
        "(mace_pnp_solve(..., denoiser=H)) or use the CNN denoiser")


def denoise(spec: DenoiserSpec, v, n_side: int):
    return make_denoiser(spec, n_side)(v)
