"""Agent-level API on the GPU (mirrors /root/reference/pkg/src/macetomo/icd.py).

``AgentWorkspace`` owns a private device plan holding one agent's stacked
operator, error sinogram and state.  ``partial_update_prox`` is one K2 pass.
The default ``schedule="raster"`` visits pixels in the reference's order
(0..n-1, one warp) and reproduces ``partial_update_prox`` pass by pass to
fp32 rounding; ``schedule="sv"`` runs the parallel super-voxel pass (same
fixed points, different visiting order).
"""

from __future__ import annotations

import numpy as np

from .engine import AgentPlan
from .geometry import ViewSubset

__all__ = ["AgentWorkspace", "ConvergenceError", "pixel_update", "partial_update_prox", "prox_solve",
           "icd_map_solve", "REFRESH_EVERY"]

REFRESH_EVERY = 50  # icd.py:29


class ConvergenceError(RuntimeError):
    """Iterative solve exhausted its budget or diverged (icd.py:32-42)."""

    def __init__(self, message, last_iterate=None, log=None):
        super().__init__(message)
        self.last_iterate = last_iterate
        self.log = log


def _default_schedule(n: int) -> str:
    return "raster" if n <= 65536 else "sv"


class AgentWorkspace:
    """One agent's private solver state on the GPU (icd.py:152-246).

    Same constructor as the reference.  ``state`` and ``error_sinogram`` are
    read back from the device as float64 copies (writes to them do not
    propagate; use ``set_state``).
    """

    def __init__(self, problem, subset: ViewSubset, n_subsets: int, sigma: float | None,
                 beta: float | None = None, state: np.ndarray | None = None, clamp_nonneg: bool = False,
                 schedule: str | None = None, device: int = 0, sv_side: int | None = None):
        if sigma is not None and sigma <= 0:
            raise ValueError("sigma must be > 0")
        self.subset = subset
        self.sigma = sigma
        self.clamp_nonneg = clamp_nonneg
        self.prior = problem.prior if beta is None else problem.prior.with_beta(beta)
        self.n = problem.geom.n_pixels
        self.schedule = schedule or _default_schedule(self.n)
        kw = {} if sv_side is None else {"sv": int(sv_side)}  # super-voxel tile side (GPU knob)
        self.plan = AgentPlan(problem.matrices, [tuple(subset.view_indices)], schedule=self.schedule, device=device,
                              **kw)
        self.plan.load_data(problem.y, problem.weights)
        self.plan.set_prior(self.prior)
        self.beta_eff = self.prior.beta / n_subsets  # icd.py:198
        self.plan.set_agent_params(0, self.beta_eff, self.inv_sigma2, clamp_nonneg)
        self.set_state(np.zeros(self.n) if state is None else state)
        self.passes = 0

    @property
    def inv_sigma2(self) -> float:
        return 0.0 if self.sigma is None else 1.0 / (self.sigma * self.sigma)

    @property
    def state(self) -> np.ndarray:
        return self.plan.get_state(0).astype(np.float64)

    @property
    def error_sinogram(self) -> np.ndarray:
        return self.plan.get_error(0).astype(np.float64)

    @property
    def curv_data(self) -> np.ndarray:
        return self.plan.get_theta2(0).astype(np.float64)

    def nnz(self) -> int:
        return int(self.plan.agent_info(0)["nnz"])

    def refresh_error(self) -> None:
        self.plan.refresh(0)

    def error_drift(self) -> float:
        """||e - (y - A z)|| / ||y - A z|| (icd.py:213-216), exact residual recomputed by K3."""
        e = self.plan.get_error(0).astype(np.float64)
        self.plan.refresh(0)
        exact = self.plan.get_error(0).astype(np.float64)
        drift = float(np.linalg.norm(e - exact)) / max(float(np.linalg.norm(exact)), 1e-300)
        return drift

    def set_state(self, x) -> None:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"state must have shape ({self.n},)")
        self.plan.set_state(0, x)

    def _run_range(self, v, s_begin, s_end) -> float:
        return float(self.plan.run_pass(0, v, 1, s_begin, s_end)[0])


def _check_target(ws: AgentWorkspace, v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (ws.n,):
        raise ValueError(f"v must have shape ({ws.n},)")
    return v


def pixel_update(ws: AgentWorkspace, s: int, v) -> float:
    """Surrogate 1-D update of pixel s (icd.py:256-269).  Needs the raster schedule."""
    if not 0 <= s < ws.n:
        raise ValueError("pixel index out of range")
    v = _check_target(ws, v)
    if ws.schedule != "raster":
        raise ValueError("pixel_update needs schedule='raster'")
    before = float(ws.plan.get_state(0)[s])
    ws._run_range(v, s, s + 1)
    return float(ws.plan.get_state(0)[s]) - before


def partial_update_prox(ws: AgentWorkspace, v) -> np.ndarray:
    """One full pass toward prox_{f_i,sigma}(v) from the remembered state (icd.py:272-283)."""
    v = _check_target(ws, v)
    ws._run_range(v, 0, ws.n)
    ws.passes += 1
    if ws.passes % REFRESH_EVERY == 0:
        ws.refresh_error()
    return ws.state


def prox_solve(ws: AgentWorkspace, v, tol: float, max_passes: int = 500) -> np.ndarray:
    """Repeat passes until sqrt(sum alpha^2)/||z|| < tol (icd.py:286-303)."""
    if tol <= 0:
        raise ValueError("tol must be > 0")
    v = _check_target(ws, v)
    for _ in range(max_passes):
        dsq = ws._run_range(v, 0, ws.n)
        ws.passes += 1
        if ws.passes % REFRESH_EVERY == 0:
            ws.refresh_error()
        z = ws.state
        if np.sqrt(dsq) / max(float(np.linalg.norm(z)), 1e-300) < tol:
            return z
    raise ConvergenceError(f"prox_solve: no convergence to {tol:g} in {max_passes} passes", last_iterate=ws.state)


CENTRAL_KAPPA = 16.0  # proximal anchor of the parallel centralized pass, x mean(theta2)


def icd_map_solve(problem, tol: float, beta: float | None = None, max_passes: int = 1000, x0=None,
                  counter=None, on_pass=None, clamp_nonneg: bool = False, schedule: str | None = None,
                  device: int = 0, kappa: float | None = None) -> np.ndarray:
    """Centralized full-data ICD without a proximal term (icd.py:306-345).

    ``schedule`` None: the reference's raster order up to 65,536 pixels, the parallel super-voxel
    pass (multi-warp tiles: one warp per 96 views) above.  Without a proximal term the tiles a
    parallel pass runs at once see each other's sinogram updates late, which diverges for the
    full-data operator (the reason for MACE's view split); the super-voxel
    schedules therefore anchor every pass at the state it starts from (target v = z, weight
    kappa x mean(theta2), default CENTRAL_KAPPA) and run at most max(4, tiles / 256) tiles at once:
    a proximal-point iteration whose fixed point (alpha = 0 with v = z) is the same MAP.  Its
    per-pass step is damped by about 1 / (1 + kappa), so the stopping test scales relnorm by
    (1 + kappa)."""
    if tol <= 0:
        raise ValueError("tol must be > 0")
    all_views = ViewSubset(0, tuple(range(problem.geom.n_views)))
    ws = AgentWorkspace(problem, all_views, 1, sigma=None, beta=beta, state=x0, clamp_nonneg=clamp_nonneg,
                        schedule=schedule, device=device)
    prox = ws.schedule != "raster"
    scale = 1.0
    if prox:
        kappa = CENTRAL_KAPPA if kappa is None else float(kappa)
        tiles = int(ws.plan.info()["n_items"])
        ws.plan.set_schedule(max(4.0, tiles / 256.0) / tiles)
        ws.plan.set_agent_params(0, ws.beta_eff, kappa * float(np.mean(ws.curv_data)), clamp_nonneg)
        scale = 1.0 + kappa
    v = np.zeros(ws.n)
    z = ws.state
    for k in range(max_passes):
        dsq = ws._run_range(z if prox else v, 0, ws.n)
        ws.passes += 1
        if ws.passes % REFRESH_EVERY == 0:
            ws.refresh_error()
        if counter is not None:
            counter.add_updates(ws.n)
        z = ws.state
        relnorm = np.sqrt(dsq) / max(float(np.linalg.norm(z)), 1e-300)
        if on_pass is not None:
            on_pass(k + 1, relnorm, z)
        if relnorm * scale < tol:
            return z
    raise ConvergenceError(f"icd_map_solve: no convergence to {tol:g} in {max_passes} passes",
                           last_iterate=ws.state)
