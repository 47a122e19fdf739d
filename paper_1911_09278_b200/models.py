"""Cost-model types (mirrors /root/reference/pkg/src/macetomo/models.py).

``PriorParams`` and ``ReconProblem`` keep the reference's fields, defaults and
validation so that problems built for the reference drop in unchanged (and
the reference's own objects are accepted by every entry point here, by duck
typing).  ``map_cost`` evaluates the global objective on the GPU (K3 +
prior-cost kernel, fp64 accumulation).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Geometry

__all__ = ["QUADRATIC", "QGGMRF", "PriorParams", "ReconProblem", "neighbor_table", "map_cost", "map_gradient",
           "likelihood_cost", "prior_cost", "book_to_reference_beta"]

QUADRATIC = "quadratic-mrf"
QGGMRF = "qggmrf"

_OFFSETS = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]  # models.py:50
_W_NORM = 4.0 + 2.0 * np.sqrt(2.0)
_RAW_W = [1 / np.sqrt(2), 1.0, 1 / np.sqrt(2), 1.0, 1.0, 1 / np.sqrt(2), 1.0, 1 / np.sqrt(2)]


@dataclass(frozen=True)
class PriorParams:
    """Prior configuration (models.py:55-90).  qGGMRF in the reference convention
    rho(d) = |d|^p / (p sx^p) * u^(q-p) / (1 + u^(q-p)), u = |d| / (T sx), 1 <= q <= p <= 2."""

    kind: str = QUADRATIC
    beta: float = 1.0
    p: float = 2.0
    q: float = 1.2
    T: float = 1.0
    sigma_x: float = 1.0
    eps_reg: float = 1e-8

    def __post_init__(self):
        if self.kind not in (QUADRATIC, QGGMRF):
            raise ValueError(f"unknown prior kind {self.kind!r}")
        if self.beta < 0:
            raise ValueError("beta must be >= 0")
        if self.kind == QGGMRF:
            if not (1.0 <= self.q <= self.p <= 2.0):
                raise ValueError("Q-GGMRF requires 1 <= q <= p <= 2")
            if self.T <= 0 or self.sigma_x <= 0:
                raise ValueError("Q-GGMRF requires T > 0 and sigma_x > 0")
        if self.eps_reg < 0:
            raise ValueError("eps_reg must be >= 0")

    def with_beta(self, beta: float) -> "PriorParams":
        return PriorParams(self.kind, beta, self.p, self.q, self.T, self.sigma_x, self.eps_reg)


def book_to_reference_beta(beta_book: float, p_book: float = 1.2, q_book: float = 2.0, T: float = 1.0) -> float:
    """BASELINE states qGGMRF as p=1.2, q=2 (book convention, potential |d|^p/(p sx^p) *
    (|d|/T sx)^(q-p)/(1+...)); the reference convention swaps p and q, so the same
    potential needs beta_ref = beta_book * q_book / (p_book * T^(q_book - p_book))."""
    return beta_book * q_book / (p_book * T ** (q_book - p_book))


@dataclass
class ReconProblem:
    """Geometry + per-view matrices + data + weights + prior (models.py:211-232)."""

    geom: Geometry
    matrices: list
    y: np.ndarray
    weights: np.ndarray
    prior: PriorParams

    def __post_init__(self):
        self.y = np.ascontiguousarray(self.y, dtype=np.float64)
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64)
        shape = (self.geom.n_views, self.geom.n_channels)
        if self.y.shape != shape or self.weights.shape != shape:
            raise ValueError(f"y and weights must have shape {shape}")
        if len(self.matrices) != self.geom.n_views:
            raise ValueError("need one sparse view matrix per view")

    @property
    def n(self) -> int:
        return self.geom.n_pixels


def neighbor_table(n_side: int):
    """(n, 8) neighbour indices (-1 off-image) and weights (models.py:93-108)."""
    n = n_side * n_side
    rows, cols = np.divmod(np.arange(n), n_side)
    idx = np.full((n, 8), -1, dtype=np.int64)
    w = np.zeros((n, 8))
    for k, (dr, dc) in enumerate(_OFFSETS):
        rr, cc = rows + dr, cols + dc
        ok = (rr >= 0) & (rr < n_side) & (cc >= 0) & (cc < n_side)
        idx[ok, k] = rr[ok] * n_side + cc[ok]
        w[ok, k] = _RAW_W[k] / _W_NORM
    return idx, w


def _costs(problem, x, beta):
    from .engine import operator_for

    op = operator_for(problem.matrices)
    params = problem.prior if beta is None else problem.prior.with_beta(beta)
    return op.cost(problem.y, problem.weights, x, params)


def map_cost(problem, x, beta: float | None = None) -> float:
    """f(x; beta) = 1/2 ||y - Ax||^2_Lambda + beta h(x) on the GPU (models.py:273-278)."""
    like, prior = _costs(problem, x, beta)
    return like + prior


def map_gradient(problem, x, beta: float | None = None):
    """grad f(x; beta) on the GPU (fp64 accumulation) and its norms [total, data, prior]: the
    stationarity certificate of a fixed point (0 at the MAP)."""
    from .engine import operator_for

    op = operator_for(problem.matrices)
    params = problem.prior if beta is None else problem.prior.with_beta(beta)
    return op.gradient(problem.y, problem.weights, x, params)


def likelihood_cost(problem, x) -> float:
    return _costs(problem, x, None)[0]


def prior_cost(problem, x, beta: float | None = None) -> float:
    return _costs(problem, x, beta)[1]
