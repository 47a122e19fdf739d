"""The reference's built-in PnP denoisers (denoisers.py:43-106) as make_denoiser returns them,
against outputs of the reference itself (tests/golden/make_denoisers.py): quadratic-prox as a dense
Cholesky solve (8 x 8) and by conjugate gradients (80 x 80, above the dense limit), boxcar at three
(size, radius) pairs including a window wider than the image border."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_1911_09278_b200.denoisers import DenoiserSpec, denoise, make_denoiser


@pytest.fixture(scope="module")
def dg():
    return dict(np.load(os.path.join(GOLDEN, "golden_denoisers.npz")))


@pytest.mark.parametrize("tag,tol", [("quadratic-prox_8_1", 1e-12), ("quadratic-prox_80_1", 1e-8),
                                     ("boxcar_13_1", 1e-13), ("boxcar_13_3", 1e-13), ("boxcar_40_2", 1e-13)])
def test_builtin_denoisers_match_reference(dg, tag, tol):
    kind = tag.rsplit("_", 2)[0]
    n_side, lam, radius = dg[f"{tag}_meta"]
    spec = DenoiserSpec(kind=kind, lam=float(lam), radius=int(radius))
    out = make_denoiser(spec, int(n_side))(dg[f"{tag}_in"])
    ref = dg[f"{tag}_out"]
    assert out.shape == ref.shape
    assert np.linalg.norm(out - ref) <= tol * np.linalg.norm(ref)
    assert np.allclose(denoise(spec, dg[f"{tag}_in"], int(n_side)), out, rtol=0, atol=0)


def test_builtin_denoiser_properties():
    # identity copies; the quadratic prox keeps constants (L 1 = 0) and contracts; boxcar keeps constants
    v = np.full(36, 3.0)
    assert np.allclose(make_denoiser(DenoiserSpec("quadratic-prox", lam=5.0), 6)(v), v)
    assert np.allclose(make_denoiser(DenoiserSpec("boxcar", radius=2), 6)(v), v)
    x = np.random.default_rng(0).standard_normal(36)
    hx = make_denoiser(DenoiserSpec("quadratic-prox", lam=5.0), 6)(x)
    assert np.linalg.norm(hx) < np.linalg.norm(x)
    with pytest.raises(ValueError):
        DenoiserSpec("median")
