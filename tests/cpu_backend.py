"""TEST INFRASTRUCTURE: a CPU stand-in for engine.AgentPlan built on the oracle.

It implements the plan interface `_run_outer` drives (load_data, stack_init, local_sum,
comm_arrays, iterate_local, iterate_finish, ...), with the oracle's float64 raster agents
doing the per-agent pass, so the multi-rank host logic of mace._run_outer (agent ownership,
all-reduce of the stack sum and norm scalars, stop test, log, gather of the stack) can be
exercised with gloo on CPU.  Never used by the product.
"""

from __future__ import annotations

import numpy as np
import torch

import oracle as O


class CpuPlan:
    def __init__(self, problem, agent_views):
        self.problem = problem
        self.views = [tuple(v) for v in agent_views]
        self.n = problem.geom.n_pixels
        self.n_side = problem.geom.n_side
        self.n_local = len(self.views)
        self.wsum = torch.zeros(self.n, dtype=torch.float64)
        self.sums = torch.zeros(5, dtype=torch.float64)
        self.log = []
        self.done = (0, 0)

    # -- setup
    def load_data(self, y, weights):
        self.y, self.lam = np.asarray(y, np.float64), np.asarray(weights, np.float64)

    def set_prior(self, prior):
        self.prior = O.Prior(prior.kind, prior.beta, prior.p, prior.q, prior.T, prior.sigma_x, prior.eps_reg)

    def set_agent_params(self, local, beta_eff, inv_sigma2, clamp=False):
        pr = O.Prior(**{**self.prior.__dict__, "beta": beta_eff})  # Agent divides by n_subsets=1 below
        sigma = 1.0 / np.sqrt(inv_sigma2)
        self.agents = [O.Agent(self.problem.matrices, self.y, self.lam, v, 1, sigma, pr, self.n_side, clamp=clamp)
                       for v in self.views]

    def set_ref(self, ref):
        self.ref = ref

    # -- stack
    def stack_init(self, w_local, n_total):
        self.W = np.zeros((self.n_local, self.n)) if w_local is None else np.array(w_local, np.float64)
        self.log, self.done = [], (0, 0)
        if n_total > 0:
            self.wbar = O.average(self.W) * self.n_local / n_total

    def local_sum(self):
        self.wsum[:] = torch.from_numpy(O.average(self.W) * self.n_local)

    def comm_arrays(self):
        return self.wsum, self.sums

    def mean_from_sum(self, n_total):
        self.wbar = self.wsum.numpy() / n_total

    def states_from(self, which):
        x = self.g if which else self.wbar
        for a in self.agents:
            a.set_state(x)

    def get_image(self, which):
        return np.array(self.g if which else self.wbar)

    def set_image(self, which, img):
        if which:
            self.g = np.array(img, np.float64)
        else:
            self.wbar = np.array(img, np.float64)

    def get_stack(self):
        return self.W.copy()

    # -- iterations
    def iterate_local(self, rho, use_g):
        if self.done[0]:  # like the device kernels: no-ops once the stop test has fired
            return
        g = self.g if use_g else self.wbar
        dsq = dw2 = wn2 = wo2 = 0.0
        for i, a in enumerate(self.agents):
            v = 2.0 * g - self.W[i]
            before = a.state.copy()
            X = a.partial_update(v)
            dsq += float(np.sum((X - before) ** 2))
            wn = O.mann_step(self.W[i], 2.0 * X - v, rho)
            dw2 += float(np.sum((wn - self.W[i]) ** 2))
            wn2 += float(np.sum(wn ** 2))
            wo2 += float(np.sum(self.W[i] ** 2))
            self.W[i] = wn
        self.local_sum()
        self.sums[:] = torch.tensor([dsq, dw2, wn2, wo2, 0.0], dtype=torch.float64)

    def iterate_finish(self, n_total, tol, it):
        if self.done[0]:
            return
        self.wbar = self.wsum.numpy() / n_total
        dsq, dw2, wn2, wo2, _ = self.sums.tolist()
        rel = np.sqrt(dw2) / max(np.sqrt(wo2), 1e-300)
        self.log.append([rel, np.sqrt(wn2), dsq, -1.0])
        if not np.isfinite(np.sqrt(wn2)):
            self.done = (2, it + 1)
        elif rel < tol:
            self.done = (1, it + 1)

    def iterate(self, iters, iter0, rho, use_g, tol, n_total, with_ref, device_denoise=False):
        for k in range(iters):
            if self.done[0]:
                break
            self.iterate_local(rho, use_g)
            self.iterate_finish(n_total, tol, iter0 + k)
        return 0.0

    def read_log(self, n):
        lg = np.array(self.log[:n], np.float64).reshape(-1, 4)
        return lg, self.done
