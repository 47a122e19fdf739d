"""Consensus-equilibrium outer loop on the GPU (mirrors /root/reference/pkg/src/macetomo/mace.py).

``mace_solve`` / ``mace_pnp_solve`` keep the reference signatures, config
validation, error behaviour and result types.  One MACE iteration

    v = (2G - I) w ;  X_i <- one ICD pass toward prox_{f_i}(v_i) ;  w <- rho (2X - v) + (1 - rho) w

runs as kernel K2 (all local agents at once, v and the Mann step fused in)
followed by K4 (fixed-order average + norms + stop test), with no host
synchronisation between iterations.  With several ranks (one process per
GPU, ``torch.distributed``), agent i lives on rank i mod world and the only
exchange per iteration is one all-reduce of the local stack sum (+4 scalars).

The small stacked-state helpers (``average``, ``reflect_G``, ``mann_step`` ...)
are the reference's host algebra, kept for API compatibility; the solver
never calls them.
"""

from __future__ import annotations

import inspect
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .denoisers import DenoiserSpec, make_denoiser
from .engine import DEFAULT_COLOURS, DEFAULT_SV, plan_for
from .geometry import partition_views
from .icd import ConvergenceError

__all__ = ["PeerComm", "MaceConfig", "MaceResult", "ConvergenceLog", "ResidualReport", "WorkerPool", "new_stack", "average",
           "consensus_G", "reflect_G", "consensus_GH", "mann_step", "mace_solve", "mace_pnp_solve",
           "equilibrium_residuals", "EquitCounter", "nrmse", "mace_solve_batch"]

CONVENTIONAL = "conventional"
PNP = "pnp"


# --------------------------------------------------------------------------- host algebra (mace.py:57-117)

def new_stack(n_subsets: int, n: int) -> np.ndarray:
    if n_subsets < 1 or n < 1:
        raise ValueError("stack dimensions must be >= 1")
    return np.zeros((n_subsets, n))


def _check_stack(stack) -> np.ndarray:
    stack = np.asarray(stack, dtype=np.float64)
    if stack.ndim != 2 or stack.shape[0] < 1:
        raise ValueError("a stacked state must be a (N, n) array with N >= 1")
    return stack


def average(stack) -> np.ndarray:
    """Balanced pairwise-tree mean in fixed order (the order K4 uses on the device)."""
    stack = _check_stack(stack)
    acc = stack.copy()
    m = acc.shape[0]
    while m > 1:
        half = m // 2
        acc[:half] += acc[half:2 * half]
        if m % 2:
            acc[half] = acc[2 * half]
            m = half + 1
        else:
            m = half
    return acc[0] / stack.shape[0]


def consensus_G(stack) -> np.ndarray:
    stack = _check_stack(stack)
    return np.broadcast_to(average(stack), stack.shape).copy()


def reflect_G(stack) -> np.ndarray:
    stack = _check_stack(stack)
    return 2.0 * average(stack)[None, :] - stack


def consensus_GH(stack, denoiser) -> np.ndarray:
    stack = _check_stack(stack)
    return np.broadcast_to(denoiser(average(stack)), stack.shape).copy()


def mann_step(w, Tw, rho: float) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    Tw = np.asarray(Tw, dtype=np.float64)
    if w.shape != Tw.shape:
        raise ValueError("w and Tw must have identical shapes")
    return rho * Tw + (1.0 - rho) * w


def nrmse(x, x_ref) -> float:
    """||x - x_ref|| / ||x_ref|| (oracle.py:341-351 of the reference)."""
    x = np.asarray(x, dtype=np.float64)
    x_ref = np.asarray(x_ref, dtype=np.float64)
    if x.shape != x_ref.shape:
        raise ValueError("shapes must match")
    scale = float(np.linalg.norm(x_ref))
    if scale == 0.0:
        raise ValueError("reference norm is zero")
    return float(np.linalg.norm(x - x_ref)) / scale


@dataclass
class EquitCounter:
    """One equit = one pass over the ROI by every one of the N agents (oracle.py:354-374)."""

    roi_voxels: int
    n_subsets: int
    updates: int = 0

    def __post_init__(self):
        if self.roi_voxels <= 0:
            raise ValueError("roi_voxels must be > 0")
        if self.n_subsets < 1:
            raise ValueError("n_subsets must be >= 1")

    def add_updates(self, count: int) -> None:
        if count < 0:
            raise ValueError("update count must be nonnegative")
        self.updates += count

    def equits(self) -> float:
        return self.updates / (self.roi_voxels * self.n_subsets)


# --------------------------------------------------------------------------- config / bookkeeping

@dataclass(frozen=True)
class MaceConfig:
    """Outer-loop configuration (mace.py:124-163) plus the GPU schedule knobs:
    ``schedule`` "sv" (parallel super-voxel passes), "sv-det" (the same, class-synchronous and
    bitwise reproducible) or "raster" (reference order),
    ``sv_side`` / ``colours`` (tile side and colour-class stride of the SV queue)."""

    n_subsets: int
    rho: float = 0.8
    sigma: float = 1.0
    mode: str = CONVENTIONAL
    beta: float | None = None
    denoiser: DenoiserSpec | None = None
    max_outer: int = 1000
    tol: float = 1e-7
    equit_accounting: bool = True
    residuals: str = "final"
    clamp_nonneg: bool = False
    schedule: str = "sv"
    sv_side: int = DEFAULT_SV
    colours: int = DEFAULT_COLOURS
    device: int = 0

    def __post_init__(self):
        if self.n_subsets < 1:
            raise ValueError("n_subsets must be >= 1")
        if not 0.0 < self.rho < 1.0:
            raise ValueError("rho must lie in (0, 1)")
        if self.sigma <= 0.0:
            raise ValueError("sigma must be > 0")
        if self.mode not in (CONVENTIONAL, PNP):
            raise ValueError(f"mode must be '{CONVENTIONAL}' or '{PNP}'")
        if self.mode == PNP and self.denoiser is None:
            raise ValueError("pnp mode requires a denoiser spec")
        if self.max_outer < 1:
            raise ValueError("max_outer must be >= 1")
        if self.tol <= 0.0:
            raise ValueError("tol must be > 0")
        if self.residuals not in ("final", "none"):
            raise ValueError("residuals must be 'final' or 'none'")
        if self.schedule not in ("sv", "raster", "sv-det"):
            raise ValueError("schedule must be 'sv', 'sv-det' or 'raster'")


class ConvergenceLog:
    """Per-iteration rows, CSV-serialisable (mace.py:166-201)."""

    COLUMNS = ("iter", "equits", "mann_update_relnorm", "r_F", "r_u", "nrmse_vs_ref", "wall_seconds")

    def __init__(self, pnp: bool = False):
        self.pnp = pnp
        self.rows: list[dict] = []

    def append(self, **kw) -> None:
        self.rows.append(kw)

    def header(self) -> tuple:
        cols = list(self.COLUMNS)
        if self.pnp:
            cols[4] = "r_H"
        return tuple(cols)

    def write_csv(self, path) -> None:
        import csv

        def fmt(v):
            return "" if v is None else repr(float(v))

        with open(path, "w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(self.header())
            for r in self.rows:
                wr.writerow([r.get("iter"), fmt(r.get("equits")), fmt(r.get("relnorm")), fmt(r.get("r_F")),
                             fmt(r.get("r_u")), fmt(r.get("nrmse")), fmt(r.get("wall"))])


@dataclass
class ResidualReport:
    mode: str
    r_F: float
    r_u: float
    per_agent: list = field(default_factory=list)


@dataclass
class MaceResult:
    image: np.ndarray
    stack: np.ndarray
    log: ConvergenceLog
    iterations: int
    converged: bool
    equits: float | None = None
    residuals: ResidualReport | None = None
    device_ms: float | None = None  # device time of the iteration loop (CUDA events)


class WorkerPool:
    """Accepted for API compatibility (mace.py:229-254).  On the GPU every local
    agent runs concurrently inside one kernel, so the worker count is unused and
    results never depend on it."""

    def __init__(self, workers: int | None = None):
        self.workers = workers

    def map(self, fn, items):
        return [fn(i) for i in items]

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# --------------------------------------------------------------------------- distributed plumbing

class _Comm:
    """Rank layout + all-reduce of the per-iteration consensus buffers (torch.distributed)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce(self, *tensors, stream=None):
        """Sum-all-reduce in place.  With `stream` (the library's stream as a torch stream) NCCL
        is enqueued behind the kernels that wrote the buffers: no host round trip per iteration."""
        if stream is None:
            for t in tensors:
                self.dist.all_reduce(t, group=self.group)
            return
        import torch

        with torch.cuda.stream(stream):
            for t in tensors:
                self.dist.all_reduce(t, group=self.group)

    def allgather_stack(self, w_loc: np.ndarray, N: int, n: int, device=None) -> np.ndarray:
        """The full (N, n) stack on every rank from each rank's agents {i : i mod world == rank}
        (float32 rows): one tensor all-gather (NCCL over NVLink when `device` is a GPU) of the
        [ceil(N / world), n] padded local blocks, then agent i = row (i // world) of rank i % world."""
        import torch

        per = -(-N // self.world)
        dev = torch.device("cpu") if device is None else device
        src = torch.from_numpy(np.ascontiguousarray(w_loc))
        blk = torch.zeros((per, n), dtype=src.dtype, device=dev)
        if len(w_loc):
            blk[: len(w_loc)] = src.to(dev)
        parts = [torch.empty_like(blk) for _ in range(self.world)]
        self.dist.all_gather(parts, blk, group=self.group)
        allp = torch.stack(parts).cpu().numpy()  # [world, per, n]
        out = np.empty((N, n), allp.dtype)
        for i in range(N):
            out[i] = allp[i % self.world, i // self.world]
        return out


def _comm_device(comm):
    """the torch device a collective of this process group runs on (its NCCL device, or the CPU
    for gloo)"""
    try:
        if comm.dist.get_backend(comm.group) == "nccl":
            import torch

            return torch.device("cuda", torch.cuda.current_device())
    except Exception:
        pass
    return None


def _f64(a: np.ndarray) -> np.ndarray:
    """float32 -> float64 result arrays (the reference returns float64) with torch's multi-threaded
    CPU conversion: a 2M-element stack converts ~5x faster than ndarray.astype."""
    if a.size < (1 << 16):
        return a.astype(np.float64)
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.float64).numpy()


def _pinned_get(plan, name, *args):
    """result read through the plan's pinned buffer when it has one (host-side test backends do not);
    the caller converts it (_f64) before the next read"""
    fn = getattr(plan, name)
    if "pinned" in inspect.signature(fn).parameters:
        return fn(*args, pinned=True)
    return fn(*args)


def _plan_stream(plan):
    """the plan's stream as a torch stream (GPU plans), None for host-side test backends"""
    ts = getattr(plan, "torch_stream", None)
    return ts() if ts is not None else None


class PeerComm(_Comm):
    """Agents on several GPUs of one node with the consensus exchanged over NVLink peer memory by
    the library's own kernels (k_peer.cuh: local tree sum pushed into every rank's symmetric
    buffer, flag, rank-ordered sum) instead of a collective; the whole MACE loop stays on the
    device.  torch.distributed's symmetric memory provides the buffers and their peer mappings."""

    def attach(self, plan):
        if getattr(plan, "_peer_comm", None) is self:
            return
        import torch
        import torch.distributed._symmetric_memory as symm

        nbytes = plan.peer_bytes(self.world)
        buf = symm.empty(nbytes, dtype=torch.uint8, device=f"cuda:{plan.device}")
        group = self.group if self.group is not None else self.dist.group.WORLD
        hdl = symm.rendezvous(buf, group)
        ptrs = np.array(list(hdl.buffer_ptrs), np.uint64)
        plan.peer_setup(self.world, self.rank, ptrs)
        plan._peer_keep = (buf, hdl)
        plan._peer_comm = self
        self.dist.barrier(group=self.group)  # every rank's flags are zero before the first exchange


def _resolve_comm(comm):
    if comm is None or comm is False:
        return None
    if comm is True:
        import torch.distributed as dist

        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
            return None
        return _Comm()
    return comm


# --------------------------------------------------------------------------- the driver (mace.py:276-365)

def _run_outer(problem, config: MaceConfig, pool, ref_image, w0, denoiser, comm=None, backend=None):
    n = problem.geom.n_pixels
    N = config.n_subsets
    subsets = partition_views(problem.geom.n_views, N)
    comm = _resolve_comm(comm)
    rank, world = (comm.rank, comm.world) if comm else (0, 1)
    local = [i for i in range(N) if i % world == rank]
    pnp = denoiser is not None
    if pnp:
        sigma, beta = np.sqrt(N) * config.sigma, 0.0  # mace.py:263-265
    else:
        sigma = config.sigma
        beta = problem.prior.beta if config.beta is None else config.beta
    views = [subsets[i].view_indices for i in local]
    if backend is None:
        # getattr: the reference's own MaceConfig (no GPU knobs) is accepted too
        plan = plan_for(problem.matrices, views, schedule=getattr(config, "schedule", "sv"),
                        sv=getattr(config, "sv_side", DEFAULT_SV), colours=getattr(config, "colours", DEFAULT_COLOURS),
                        device=getattr(config, "device", 0))
    else:
        plan = backend(problem, views)
    plan.load_data(problem.y, problem.weights)
    plan.set_prior(problem.prior)
    plan.set_agent_params(-1, beta / N, 1.0 / (sigma * sigma), config.clamp_nonneg)

    if w0 is not None:
        w0 = _check_stack(w0)
        if w0.shape != (N, n):
            raise ValueError(f"w0 must have shape ({N}, {n})")
        w_local = np.ascontiguousarray(w0[local], np.float32)
    else:
        w_local = None
    peer = isinstance(comm, PeerComm)
    if comm is None:
        plan.stack_init(w_local, N)
    elif peer:
        comm.attach(plan)
        plan.stack_init(w_local, 0)
        plan.peer_mean(N)
    else:
        plan.stack_init(w_local, 0)
        plan.local_sum()
        comm.allreduce(*plan.comm_arrays()[:1], stream=_plan_stream(plan))
        plan.mean_from_sum(N)
    device_g = pnp and getattr(denoiser, "device_apply", None) is not None
    if pnp:
        _apply_denoiser(plan, denoiser)
        plan.states_from(1)  # X0 = H(average(w0)), mace.py:286
    else:
        plan.states_from(0)  # X0 = average(w0)
    ref32 = None if ref_image is None else np.ascontiguousarray(ref_image, np.float32)
    ref_norm = None if ref_image is None else float(np.linalg.norm(np.asarray(ref_image, np.float64)))
    if ref_image is not None and ref_norm == 0.0:
        raise ValueError("reference norm is zero")
    plan.set_ref(ref32 if (not pnp and comm is None) else None)

    log = ConvergenceLog(pnp=pnp)
    counter = EquitCounter(n, N) if config.equit_accounting else None
    t0 = time.perf_counter()
    device_ms = 0.0
    rows = []  # (relnorm, nrmse, wall)
    done = (0, 0)
    it = 0
    if peer and pnp and not device_g:
        raise ValueError("the peer-memory consensus needs a device denoiser (CnnDenoiser) or none")
    host_loop = (comm is not None and not peer) or (pnp and not device_g)
    if not host_loop:
        chunk = config.max_outer
        while it < config.max_outer and done[0] == 0:
            k = min(chunk, config.max_outer - it)
            in_loop = pnp and hasattr(denoiser, "_load")  # the K5 CNN: H inside the device loop
            host_nr = ref_image is not None and (pnp or peer)  # NRMSE from the image on the host
            if host_nr or (pnp and not in_loop):  # per-iteration host step
                k = 1
            if in_loop:
                denoiser._load(plan)
            if peer:
                ms = plan.iterate_peer(k, it, config.rho, pnp, config.tol, N, device_denoise=in_loop)
            else:
                ms = plan.iterate(k, it, config.rho, pnp, config.tol, N, ref32 is not None, device_denoise=in_loop)
            device_ms += ms
            if pnp and not in_loop:
                _apply_denoiser(plan, denoiser)
            it += k
            lg, done = plan.read_log(it)
            wall = time.perf_counter() - t0
            lim = it if done[0] == 0 else (done[1] if done[0] == 1 else done[1] - 1)
            for j in range(len(rows), lim):
                nr = None
                if ref_image is not None:  # the device log holds the NRMSE only for a single context
                    nr = nrmse(plan.get_image(1 if pnp else 0), ref_image) if host_nr else lg[j, 3]
                rows.append((lg[j, 0], nr, wall * (j + 1) / it))
    else:
        # multi-rank (or host-denoiser) loop: K2 + local sum -> all-reduce on the library stream ->
        # finish; the log is read back only every 50 iterations unless a per-iteration host step
        # (host denoiser, NRMSE against ref_image) needs it.  After the stop test fires, the
        # device `done` flag turns the remaining launches into no-ops.
        stream = _plan_stream(plan)
        per_iter_host = ref_image is not None or (pnp and not device_g)
        k = 0
        if comm is not None and stream is not None and not per_iter_host and GRAPH_BLOCK > 0:
            # whole blocks of GRAPH_BLOCK iterations as one CUDA graph (captured once, replayed): one
            # host call per block instead of ~4 launches and a collective per iteration
            plan.reserve_log(config.max_outer)
            graph = None
            while k + GRAPH_BLOCK <= config.max_outer:
                plan.set_iter(k)
                if graph is None:
                    graph = _capture_block(plan, comm, stream, GRAPH_BLOCK, config.rho, pnp, N, config.tol,
                                           denoiser)
                _replay(graph, stream)
                plan.add_passes(GRAPH_BLOCK)
                k += GRAPH_BLOCK
                lg, done = plan.read_log(k)
                it = k
                wall = time.perf_counter() - t0
                lim = k if done[0] == 0 else (done[1] if done[0] == 1 else done[1] - 1)
                for j in range(len(rows), lim):
                    rows.append((lg[j, 0], None, wall * (j + 1) / k))
                if done[0]:
                    break
        while k < config.max_outer and done[0] == 0:
            plan.iterate_local(config.rho, pnp)
            if comm is not None:
                comm.allreduce(*plan.comm_arrays(), stream=stream)
            plan.iterate_finish(N, config.tol, k)
            if pnp:
                _apply_denoiser(plan, denoiser)
            k += 1
            if not (per_iter_host or k == config.max_outer or k % 50 == 0):
                continue
            lg, done = plan.read_log(k)
            it = k
            wall = time.perf_counter() - t0
            lim = k if done[0] == 0 else (done[1] if done[0] == 1 else done[1] - 1)
            for j in range(len(rows), lim):
                est = None
                if ref_image is not None:
                    est = nrmse(plan.get_image(1 if pnp else 0), ref_image)
                rows.append((lg[j, 0], est, wall * (j + 1) / k))
            if done[0]:
                break
    if done[0] == 2:
        raise ConvergenceError(
            f"MACE diverged at iteration {done[1]}: the partial-update map is expansive for this sigma "
            "(reduce sigma)", last_iterate=None, log=_fill_log(log, rows, counter, N, n))
    iterations = len(rows)
    converged = done[0] == 1
    _fill_log(log, rows, counter, N, n)
    image = _f64(_pinned_get(plan, "get_image", 1 if pnp else 0))
    if comm is None:
        stack = _f64(_pinned_get(plan, "get_stack").reshape(len(local), n))
    else:
        w_loc = np.array(_pinned_get(plan, "get_stack").reshape(len(local), n))  # a copy of the pinned view
        stack = _f64(comm.allgather_stack(w_loc, N, n, device=_comm_device(comm)))
    result = MaceResult(image=image, stack=stack, log=log, iterations=iterations, converged=converged,
                        equits=None if counter is None else counter.equits(), device_ms=device_ms)
    if config.residuals == "final":
        result.residuals = equilibrium_residuals(problem, config, stack, denoiser=denoiser)
        if log.rows:
            log.rows[-1]["r_F"] = result.residuals.r_F
            log.rows[-1]["r_u"] = result.residuals.r_u
    if not converged:
        raise ConvergenceError(f"MACE: Mann update relnorm did not reach {config.tol:g} in {config.max_outer} "
                               "iterations", last_iterate=result, log=log)
    return result


# iterations per captured CUDA graph in the multi-rank loop (0: launch every iteration from the host);
# 50 = the error-refresh period, so every replay carries exactly one refresh at the same place
GRAPH_BLOCK = int(os.environ.get("MACE_GRAPH_BLOCK", "50"))


def _capture_block(plan, comm, stream, G, rho, pnp, N, tol, denoiser):
    """G multi-rank MACE iterations (K2 + local sum -> all-reduce -> finish [-> K5]) captured into a
    CUDA graph on the library stream; the log rows come from the device iteration counter.  The
    capture executes nothing, so the host pass count it advanced is taken back."""
    import torch

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        for _ in range(G):
            plan.iterate_local(rho, pnp)
            comm.allreduce(*plan.comm_arrays(), stream=stream)
            plan.iterate_finish(N, tol, -1)
            if pnp:
                _apply_denoiser(plan, denoiser)
    plan.add_passes(-G)
    return g


def _replay(graph, stream):
    import torch

    with torch.cuda.stream(stream):
        graph.replay()


def _fill_log(log, rows, counter, N, n):
    log.rows.clear()
    if counter is not None:
        counter.updates = 0
    for j, (rel, nr, wall) in enumerate(rows):
        if counter is not None:
            counter.add_updates(N * n)
        log.append(iter=j + 1, equits=None if counter is None else counter.equits(), relnorm=float(rel), r_F=None,
                   r_u=None, nrmse=None if nr is None else float(nr), wall=wall)
    return log


def _apply_denoiser(plan, denoiser):
    dev = getattr(denoiser, "device_apply", None)
    if dev is not None:
        dev(plan)  # reads wbar, writes g on the device
        return
    wbar = plan.get_image(0).astype(np.float64)
    h = np.asarray(denoiser(wbar), dtype=np.float64)
    if h.shape != wbar.shape:
        raise ValueError("denoiser must map a length-n image to a length-n image")
    plan.set_image(1, h)


def mace_solve(problem, config: MaceConfig, pool: WorkerPool | None = None, ref_image=None, w0=None,
               comm=None, _backend=None) -> MaceResult:
    """Partial-update MACE with the conventional prior (mace.py:368-382).  Converges to
    the MAP image of the full-data objective; returns the component average.

    ``comm``: None (single process), True (use the initialised default torch.distributed
    group: agent i on rank i mod world), or a communicator object.  ``_backend`` is a test
    hook replacing the device plan (the CPU tests of the multi-rank logic use it)."""
    if config.mode != CONVENTIONAL:
        raise ValueError("mace_solve requires mode='conventional'")
    return _run_outer(problem, config, pool, ref_image, w0, denoiser=None, comm=comm, backend=_backend)


def mace_pnp_solve(problem, config: MaceConfig, pool: WorkerPool | None = None, ref_image=None, w0=None,
                   denoiser=None, comm=None, _backend=None) -> MaceResult:
    """MACE with a PnP denoiser prior (mace.py:385-404): agents carry only data terms at
    sqrt(N) sigma; H acts once per iteration on the average; returns H(mean w)."""
    if config.mode != PNP:
        raise ValueError("mace_pnp_solve requires mode='pnp'")
    if denoiser is None:
        denoiser = make_denoiser(config.denoiser, problem.geom.n_side)
    return _run_outer(problem, config, pool, ref_image, w0, denoiser=denoiser, comm=comm, backend=_backend)


def mace_solve_batch(problems, config: MaceConfig) -> list:
    """Independent conventional MACE solves of several slices that share one scan geometry
    (BASELINE config 4: 64 slices, N view agents, one operator).  Equivalent to
    ``[mace_solve(p, config) for p in problems]`` except that the stop test uses the Mann
    relnorm of the whole batch.  On the GPU the slices of an agent run as concurrent agents
    on the same super-voxel tile, so each tile's A columns stream from HBM once per
    iteration for all slices.  Returns one MaceResult per slice (the log is shared); raises
    ConvergenceError (``last_iterate`` = that list) when the budget runs out."""
    problems = list(problems)
    if not problems:
        raise ValueError("need at least one problem")
    if config.mode != CONVENTIONAL:
        raise ValueError("mace_solve_batch requires mode='conventional'")
    p0 = problems[0]
    for p in problems[1:]:
        if p.matrices is not p0.matrices or p.y.shape != p0.y.shape:
            raise ValueError("batched slices must share the matrices object and geometry")
        if p.prior != p0.prior:
            raise ValueError("batched slices must share the prior")
    S, N, n = len(problems), config.n_subsets, p0.geom.n_pixels
    subsets = partition_views(p0.geom.n_views, N)
    plan = plan_for(p0.matrices, [s.view_indices for s in subsets], schedule="sv",
                    sv=getattr(config, "sv_side", DEFAULT_SV), colours=getattr(config, "colours", DEFAULT_COLOURS),
                    device=getattr(config, "device", 0), n_slices=S)
    beta = p0.prior.beta if config.beta is None else config.beta
    plan.load_data([p.y for p in problems], [p.weights for p in problems])
    plan.set_prior(p0.prior)
    plan.set_agent_params(-1, beta / N, 1.0 / (config.sigma * config.sigma), config.clamp_nonneg)
    plan.stack_init(None, N)
    plan.states_from(0)
    plan.set_ref(None)
    t0 = time.perf_counter()
    ms = plan.iterate(config.max_outer, 0, config.rho, False, config.tol, N, False)
    lg, done = plan.read_log(config.max_outer)
    wall = time.perf_counter() - t0
    if done[0] == 2:
        raise ConvergenceError(f"MACE diverged at iteration {done[1]} (reduce sigma)", last_iterate=None)
    iters = done[1] if done[0] == 1 else config.max_outer
    images = _f64(plan.get_image(0, pinned=True).reshape(S, n))
    stacks = _f64(plan.get_stack(pinned=True).reshape(S, N, n))
    log = ConvergenceLog()
    counter = EquitCounter(n, N)
    _fill_log(log, [(lg[j, 0], None, wall * (j + 1) / max(iters, 1)) for j in range(iters)], counter, N, n)
    results = [MaceResult(image=images[s], stack=stacks[s], log=log, iterations=iters, converged=done[0] == 1,
                          equits=counter.equits(), device_ms=ms) for s in range(S)]
    if done[0] != 1:
        raise ConvergenceError(f"MACE batch: relnorm did not reach {config.tol:g} in {config.max_outer} iterations",
                               last_iterate=results, log=log)
    return results


# float32 state: the relative update of a proximal pass bottoms out near 1e-7 (rounding of theta1 and of
# z itself), so the equilibrium check's prox solves stop at max(prox_tol, PROX_TOL_FP32) instead of the
# reference's float64 1e-9 (mace.py:411); r_F is then resolved to ~1e-6 (tests/test_gpu_residuals.py)
PROX_TOL_FP32 = 1e-6


def equilibrium_residuals(problem, config: MaceConfig, w, prox_tol: float = 1e-9, denoiser=None) -> ResidualReport:
    """Equilibrium check of a stacked state (mace.py:407-454).  Conventional: x_hat = mean w,
    u_i = x_hat - w_i, r_F = max_i ||F_i(x_hat + u_i; sigma) - x_hat|| / ||x_hat|| with F_i the
    converged proximal map of agent i, r_u = ||sum_i u_i|| / ||x_hat||.  PnP: x_hat = H(mean w),
    t_i = x_hat - w_i, agents at sqrt(N) sigma and beta 0, r_H = ||H(x_hat + (mean w - x_hat)) -
    x_hat|| / ||x_hat||.  All N proximal maps are solved at once on the GPU, by the context of
    the agents' layouts (cached per scan: the one mace_solve used), raster order up to 65,536
    pixels (as AgentWorkspace) and super-voxel passes beyond."""
    w = _check_stack(w)
    N = config.n_subsets
    subsets = partition_views(problem.geom.n_views, N)
    if w.shape[0] != N:
        raise ValueError(f"w must have {N} rows")
    w_bar = average(w)
    if config.mode == PNP:
        if denoiser is None:
            denoiser = make_denoiser(config.denoiser, problem.geom.n_side)
        x_hat = np.asarray(denoiser(w_bar), np.float64)
        sigma, beta = np.sqrt(N) * config.sigma, 0.0
        seconds = x_hat - w
        aux = float(np.linalg.norm(np.asarray(denoiser(x_hat + (w_bar - x_hat)), np.float64) - x_hat))
    else:
        x_hat = w_bar
        sigma = config.sigma
        beta = problem.prior.beta if config.beta is None else config.beta
        seconds = x_hat - w
        aux = float(np.linalg.norm(seconds.sum(axis=0)))
    scale = max(float(np.linalg.norm(x_hat)), 1e-300)
    n = problem.geom.n_pixels
    from .icd import _default_schedule

    plan = plan_for(problem.matrices, [s.view_indices for s in subsets], schedule=_default_schedule(n),
                    sv=getattr(config, "sv_side", DEFAULT_SV), colours=getattr(config, "colours", DEFAULT_COLOURS),
                    device=getattr(config, "device", 0))
    plan.load_data(problem.y, problem.weights)
    plan.set_prior(problem.prior)
    plan.set_agent_params(-1, beta / N, 1.0 / (sigma * sigma), getattr(config, "clamp_nonneg", False))
    tol = max(prox_tol, PROX_TOL_FP32)
    passes, rel = plan.prox_all(x_hat[None, :] + seconds, x_hat, tol, max_passes=500)
    if not np.all(rel < tol):
        raise ConvergenceError(f"equilibrium_residuals: proximal maps not converged to {tol:g} in {passes} passes "
                               f"(worst {float(rel.max()):.2e})")
    per_agent = [float(np.linalg.norm(plan.get_state(i).astype(np.float64) - x_hat)) / scale for i in range(N)]
    return ResidualReport(mode=config.mode, r_F=max(per_agent), r_u=aux / scale, per_agent=per_agent)
