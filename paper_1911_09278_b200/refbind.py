"""Bind the reference package (macetomo) to the B200 library.

Two levels, see INTEGRATION.md:

* ``sweep`` has the exact signature and semantics of the reference's numba
  ``_sweep`` (pkg/src/macetomo/icd.py:67-139): float64 arrays, raster order,
  mutates ``z`` and ``e`` in place, returns sum(alpha^2).  It runs on the GPU
  through ``mace_sweep_f64``.  ``install(macetomo)`` rebinds
  ``macetomo.icd._sweep`` (resolved at call time by ``_run_range``,
  icd.py:222-246), so every reference agent pass runs on the B200.
* ``install_solvers(macetomo)`` replaces ``mace_solve`` / ``mace_pnp_solve``
  with this package's device-resident solvers (the fast path).
"""

from __future__ import annotations

import numpy as np

from . import _native as N


def _f64(a, writable=False):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        if writable:
            raise TypeError("z and e must be C-contiguous float64 arrays (they are updated in place)")
        a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _i64(a):
    return a if (isinstance(a, np.ndarray) and a.dtype == np.int64 and a.flags.c_contiguous) else \
        np.ascontiguousarray(a, dtype=np.int64)


def sweep(z, v, e, col_ptr, row_idx, a_val, lam, curv_data, nbr_idx, nbr_w, beta_eff, eps_reg, inv_sigma2,
          quad_prior, p, q, T, sx, clamp, s_begin, s_end):
    """Drop-in for macetomo.icd._sweep (same 21 arguments, same effects)."""
    z = _f64(z, True)
    e = _f64(e, True)
    v, a_val, lam, curv_data, nbr_w = (_f64(x) for x in (v, a_val, lam, curv_data, nbr_w))
    col_ptr, row_idx, nbr_idx = _i64(col_ptr), _i64(row_idx), _i64(nbr_idx)
    n = z.shape[0]
    dsq = np.zeros(1)
    N.check(N.lib().mace_sweep_f64(
        N.ptr(z), N.ptr(v), N.ptr(e), N.ptr(col_ptr), N.ptr(row_idx), N.ptr(a_val), N.ptr(lam), N.ptr(curv_data),
        N.ptr(nbr_idx), N.ptr(nbr_w), float(beta_eff), float(eps_reg), float(inv_sigma2), int(bool(quad_prior)),
        float(p), float(q), float(T), float(sx), int(bool(clamp)), int(s_begin), int(s_end), int(n),
        int(e.shape[0]), N.ptr(dsq)), "mace_sweep_f64")
    return float(dsq[0])


def install(macetomo_pkg):
    """Rebind the reference's compiled plug point to the B200 kernel."""
    macetomo_pkg.icd._sweep = sweep
    return macetomo_pkg


def install_solvers(macetomo_pkg):
    """Replace the reference's MACE entry points with the device-resident solvers."""
    from . import mace

    for mod in (macetomo_pkg, macetomo_pkg.mace):
        mod.mace_solve = mace.mace_solve
        mod.mace_pnp_solve = mace.mace_pnp_solve
    return macetomo_pkg
