"""Shared fixtures.  ``-m "not gpu"`` runs here (no GPU); ``-m gpu`` on a B200."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(GOLDEN, "golden_small.npz")))


def unpack_views(g, prefix, n_views, n_channels, n_pixels):
    """Rebuild per-view CSR blocks from a packed fixture."""
    from oracle import ViewCSR

    rp_all = g[f"{prefix}_row_ptr"]
    cols, lens = g[f"{prefix}_cols"], g[f"{prefix}_lens"]
    nnz = g[f"{prefix}_nnz_per_view"]
    out, off = [], 0
    for k in range(n_views):
        rp = rp_all[k * (n_channels + 1):(k + 1) * (n_channels + 1)]
        out.append(ViewCSR(rp.copy(), cols[off:off + nnz[k]].copy(), lens[off:off + nnz[k]].copy(),
                           n_channels, n_pixels))
        off += nnz[k]
    return out


def small_problem(seed, n_side, n_views, n_channels):
    """Same recipe as the reference's tests/conftest.py:17-32 (geometry + random y/weights)."""
    from oracle import build_system_matrix

    rng = np.random.default_rng(seed)
    mats = build_system_matrix(n_side, 1.0, n_views, n_channels, n_side / n_channels * 1.1)
    y = rng.standard_normal((n_views, n_channels))
    w = 0.5 + rng.random((n_views, n_channels))
    return mats, y, w


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
