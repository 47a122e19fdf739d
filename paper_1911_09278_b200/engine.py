"""Device plans: native contexts holding the operator, the data and the agents.

``DeviceOperator`` — one GPU context with the full-data CSR (kernel K3) for
forward projection and costs.  ``AgentPlan`` — a context with the per-agent
layouts (kernel K1 data) for a given partition, used by the MACE driver and
by ``AgentWorkspace``.  Plans are cached per matrices object so repeated
solves on the same scan (the benchmark's end-to-end steps) only move the
sinogram and the result across PCIe.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from collections import OrderedDict

import numpy as np

from . import _native as N
from .geometry import global_csr

SCHEDULES = {"sv": 0, "raster": 1, "sv-det": 0}  # sv-det: deterministic class-synchronous super-voxel passes
SV_SIDES = (2, 4, 6, 8, 12, 16)  # tile sides compiled into k_icd_sv
DEFAULT_SV = int(os.environ.get("MACE_SV", "8"))
DEFAULT_COLOURS = int(os.environ.get("MACE_COLOURS", "4"))
DEFAULT_CONCURRENCY = float(os.environ.get("MACE_SV_CONCURRENCY", str(1.0 / 16.0)))


def _n_side_of(matrices) -> int:
    n = matrices[0].n_pixels
    s = int(math.isqrt(n))
    if s * s != n:
        raise ValueError("image must be square")
    return s


class _Context:
    """Owns one native context (destroyed with the object)."""

    def __init__(self, device: int = 0):
        self.L = N.lib()
        h = ctypes.c_void_p()
        N.check(self.L.mace_ctx_create(int(device), ctypes.byref(h)), "ctx_create")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.mace_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name, *args):
        N.check(getattr(self.L, name)(self.h, *args), name)

    def info(self):
        buf = np.zeros(10, np.int64)
        self.call("mace_ctx_info", N.ptr(buf))
        return dict(zip(["nnz", "n_items", "NV", "sv_smem", "sv_grid", "num_sms", "passes", "S", "weighted"],
                        buf.tolist()))

    def load_matrix(self, matrices):
        self.n_side = _n_side_of(matrices)
        self.n_views = len(matrices)
        self.n_ch = matrices[0].n_channels
        self.n = self.n_side * self.n_side
        rp, cols, vals = global_csr(matrices)
        self.nnz = int(rp[-1])
        self.call("mace_load_matrix", self.n_side, self.n_views, self.n_ch, N.ptr(rp), N.ptr(cols), N.ptr(vals))

    def set_prior(self, prior):
        kind = 0 if prior.kind == "quadratic-mrf" else 1
        self.call("mace_set_prior", kind, float(prior.p), float(prior.q), float(prior.T), float(prior.sigma_x),
                  float(prior.eps_reg))


class DeviceOperator(_Context):
    """Forward projector and cost evaluator for one system matrix."""

    def __init__(self, matrices, device: int = 0):
        super().__init__(device)
        self.load_matrix(matrices)
        self._data_key = None

    def forward_project(self, x) -> np.ndarray:
        x = N.f32(x)
        out = np.empty((self.n_views, self.n_ch), np.float32)
        self.call("mace_forward_project", N.ptr(x), N.ptr(out))
        return out

    def back_project(self, sino) -> np.ndarray:
        s32 = N.f32(sino)
        out = np.empty(self.n_side * self.n_side, np.float64)
        self.call("mace_back_project", N.ptr(s32), N.ptr(out))
        return out

    def load_data(self, y, weights):
        y32, w32 = N.f32(y), N.f32(weights)
        self.call("mace_load_data", N.ptr(y32), N.ptr(w32))

    def cost(self, y, weights, x, prior) -> tuple[float, float]:
        self.load_data(y, weights)
        self.set_prior(prior)
        x = N.f32(x)
        like, pri = ctypes.c_double(), ctypes.c_double()
        self.call("mace_cost", N.ptr(x), float(prior.beta), ctypes.byref(like), ctypes.byref(pri))
        return like.value, pri.value

    def gradient(self, y, weights, x, prior, want_grad=True):
        """grad f(x) (fp64, length n or None) and [|grad|, |data part|, |prior part|]"""
        self.load_data(y, weights)
        self.set_prior(prior)
        x = N.f32(x)
        norms = np.zeros(3, np.float64)
        g = np.zeros(x.shape[0], np.float64) if want_grad else None
        self.call("mace_gradient", N.ptr(x), float(prior.beta), N.ptr(g), N.ptr(norms))
        return g, norms


_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_CACHE_LOCK = threading.Lock()
_CACHE_MAX = int(os.environ.get("MACE_PLAN_CACHE", "6"))


def _cached(key, factory, keepalive):
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0] is keepalive:
            _CACHE.move_to_end(key)
            return hit[1]
    obj = factory()
    with _CACHE_LOCK:
        _CACHE[key] = (keepalive, obj)
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    return obj


def clear_cache():
    with _CACHE_LOCK:
        _CACHE.clear()


def operator_for(matrices, device: int = 0) -> DeviceOperator:
    return _cached(("op", id(matrices), device), lambda: DeviceOperator(matrices, device), matrices)


SV_MAX_VIEWS = 16 * 96  # lane-per-view layout: up to 16 view chunks (warps) of 3 x 32 views per tile


class AgentPlan(_Context):
    """Context with the layouts of ``agent_views`` (one tuple of view indices per local agent)."""

    def __init__(self, matrices, agent_views, schedule: str = "sv", sv: int = DEFAULT_SV,
                 colours: int = DEFAULT_COLOURS, device: int = 0, n_slices: int = 1):
        super().__init__(device)
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {sorted(SCHEDULES)}")
        self.load_matrix(matrices)
        self.agent_views = [tuple(int(v) for v in vs) for vs in agent_views]
        if schedule in ("sv", "sv-det") and max(len(v) for v in self.agent_views) > SV_MAX_VIEWS and int(n_slices) == 1:
            # the lane-per-view super-voxel layout holds at most 16 chunks of 96 views per agent
            # (multi-warp tiles); agents with more views run the raster pass
            schedule = "raster"
        self.schedule = schedule
        det = schedule == "sv-det"
        counts = np.array([len(v) for v in self.agent_views], np.int32)
        flat = np.array([v for vs in self.agent_views for v in vs], np.int32)
        sv_eff = sv
        if schedule in ("sv", "sv-det"):
            lim = min(sv, self.n_side + (self.n_side & 1))
            sv_eff = max([s for s in SV_SIDES if s <= max(lim, 2)])
        self.n_slices = int(n_slices)
        self.call("mace_setup_agents", len(self.agent_views), N.ptr(counts), N.ptr(flat), SCHEDULES[schedule],
                  int(sv_eff), int(colours), 0, self.n_slices)
        # local (virtual) agents: slice-major, index = slice * n_agents + agent
        self.n_agents = len(self.agent_views)
        self.n_local = self.n_agents * self.n_slices
        self.set_schedule(DEFAULT_CONCURRENCY, int(os.environ.get("MACE_SV_MAX_WARPS", "0")))
        if det:
            self.call("mace_set_deterministic", 1)
        # weighted records (a sqrt(lambda), k_sv.cuh) where the data allow them; MACE_WEIGHTED=0 forbids
        self.set_weighting(os.environ.get("MACE_WEIGHTED", "1") != "0")

    def set_weighting(self, allow: bool):
        """Allow or forbid K2's weighted records from the next ``load_data`` on."""
        self.call("mace_set_weighting", int(bool(allow)))

    def agent_info(self, a):
        buf = np.zeros(8, np.int64)
        self.call("mace_agent_info", int(a), N.ptr(buf))
        return dict(zip(["nnz", "entries", "R", "max_col", "wcap", "n_sv", "duplicates", "ctx_wcap"],
                        buf.tolist()))

    def load_data(self, y, weights):
        """y / weights ([n_slices x] n_views x n_ch, any float dtype; or, for a batch, sequences of
        n_slices per-slice arrays) -> pinned float32 staging -> device."""
        rows = self.n_views * self.n_ch * getattr(self, "n_slices", 1)
        if getattr(self, "_pin", None) is None:
            p = ctypes.c_void_p()
            N.check(self.L.mace_host_alloc(2 * rows * 4, ctypes.byref(p)), "host_alloc")
            self._pin = p
            self._pin_arr = np.ctypeslib.as_array((ctypes.c_float * (2 * rows)).from_address(p.value))
        else:  # the previous load's copies may still be reading the staging buffer
            self.call("mace_stage_wait")
        for k, src in enumerate((y, weights)):
            dst = self._pin_arr[k * rows:(k + 1) * rows]
            if isinstance(src, (list, tuple)):  # per-slice arrays straight into their staging slots
                per = rows // max(len(src), 1)
                if len(src) * per != rows:
                    raise ValueError("need one sinogram per slice")
                for j, a in enumerate(src):
                    _convert_into(dst[j * per:(j + 1) * per], np.asarray(a).reshape(-1))
            else:
                _convert_into(dst, np.asarray(src).reshape(-1))
        self.call("mace_load_data", ctypes.c_void_p(self._pin.value), ctypes.c_void_p(self._pin.value + rows * 4))

    def _pinned_out(self, count) -> np.ndarray:
        """a pinned float32 host buffer for results (D2H at full PCIe rate); valid until the next call"""
        if getattr(self, "_pout", None) is None or self._pout_n < count:
            self._free_pout()
            p = ctypes.c_void_p()
            N.check(self.L.mace_host_alloc(count * 4, ctypes.byref(p)), "host_alloc")
            self._pout, self._pout_n = p, count
            self._pout_arr = np.ctypeslib.as_array((ctypes.c_float * count).from_address(p.value))
        return self._pout_arr[:count]

    def _free_pout(self):
        if getattr(self, "_pout", None) is not None:
            if getattr(self, "h", None):
                self.L.mace_sync(self.h)
            self.L.mace_host_free(self._pout)
            self._pout = None

    def close(self):
        self._free_pout()
        if getattr(self, "_pin", None) is not None:
            if getattr(self, "h", None):
                self.L.mace_sync(self.h)
            self.L.mace_host_free(self._pin)
            self._pin = None
        super().close()

    def set_schedule(self, concurrency=DEFAULT_CONCURRENCY, max_warps=0):
        self.call("mace_set_schedule", float(concurrency), int(max_warps))

    def set_agent_groups(self, group: int):
        """Super-voxel queue in groups of `group` agents (0: all at once); see mace_set_agent_groups."""
        self.call("mace_set_agent_groups", int(group))

    def set_agent_params(self, local, beta_eff, inv_sigma2, clamp=False):
        self.call("mace_set_agent_params", int(local), float(beta_eff), float(inv_sigma2), int(bool(clamp)))

    def set_state(self, local, x):
        x = N.f32(x)
        self.call("mace_set_state", int(local), N.ptr(x))

    def get_state(self, local) -> np.ndarray:
        out = np.empty(self.n, np.float32)
        self.call("mace_get_state", int(local), N.ptr(out))
        return out

    def get_error(self, local) -> np.ndarray:
        R = len(self.agent_views[local]) * self.n_ch
        out = np.empty(R, np.float32)
        self.call("mace_get_error", int(local), N.ptr(out))
        return out

    def get_theta2(self, local) -> np.ndarray:
        out = np.empty(self.n, np.float32)
        self.call("mace_get_theta2", int(local), N.ptr(out))
        return out

    def get_batch_consts(self, local) -> np.ndarray:
        """(n_sv, batches, 16) float32: k_sv_consts' theta2 x4 and cross terms of each 4-pixel batch"""
        cnt = ctypes.c_int64(0)
        self.call("mace_get_batch_consts", int(local), None, ctypes.byref(cnt))
        out = np.empty(cnt.value, np.float32)
        self.call("mace_get_batch_consts", int(local), N.ptr(out), ctypes.byref(cnt))
        info = self.agent_info(local % self.n_agents)
        return out.reshape(info["n_sv"], -1, 16)

    def refresh(self, local=-1):
        self.call("mace_refresh", int(local))

    def prox_all(self, v, x0, tol, max_passes=500):
        """Every local agent's proximal map at once: states start at x0, targets v (n_local, n);
        passes until each agent's sqrt(sum alpha^2)/||z|| < tol.  Returns (passes, rel[n_local]);
        the solutions are the agents' states."""
        v = N.f32(np.asarray(v).reshape(self.n_local, self.n))
        x0 = N.f32(x0)
        passes = ctypes.c_int(0)
        rel = np.zeros(self.n_local, np.float64)
        self.call("mace_prox_all", N.ptr(v), N.ptr(x0), int(max_passes), float(tol), ctypes.byref(passes),
                  N.ptr(rel))
        return passes.value, rel

    def run_pass(self, local, v, n_passes=1, s_begin=0, s_end=-1) -> np.ndarray:
        v = N.f32(v)
        dsq = np.zeros(n_passes, np.float64)
        self.call("mace_pass", int(local), N.ptr(v), int(n_passes), int(s_begin), int(s_end), N.ptr(dsq))
        return dsq


    # ---------------------------------------------------------------- MACE outer loop
    def stack_init(self, w_local, n_total):
        w = None if w_local is None else N.f32(w_local)
        self.call("mace_stack_init", N.ptr(w), int(n_total))

    def local_sum(self):
        self.call("mace_local_sum")

    def mean_from_sum(self, n_total):
        self.call("mace_mean_from_sum", int(n_total))

    def comm_arrays(self):
        """(stack sum [n] float32, norm sums [5] float64) as torch CUDA tensors over the context's
        buffers.  No host synchronisation: reduce them on `torch_stream()`, which orders the
        collective after the kernels that produced them and before the ones that consume them."""
        import torch

        if getattr(self, "_comm_t", None) is None:
            wsum, sums = ctypes.c_void_p(), ctypes.c_void_p()
            self.call("mace_comm_buffers", ctypes.byref(wsum), ctypes.byref(sums))
            self._comm_t = (torch.as_tensor(_DevArray(wsum.value, (self.n,), "<f4"), device=f"cuda:{self.device}"),
                            torch.as_tensor(_DevArray(sums.value, (5,), "<f8"), device=f"cuda:{self.device}"))
        return self._comm_t

    def torch_stream(self):
        """The library stream as a torch stream (collectives enqueued on it need no host sync)."""
        import torch

        if getattr(self, "_tstream", None) is None:
            s = ctypes.c_void_p()
            self.call("mace_ctx_stream", ctypes.byref(s))
            self._tstream = torch.cuda.ExternalStream(s.value, device=f"cuda:{self.device}")
        return self._tstream

    def states_from(self, which):
        self.call("mace_states_from", int(which))

    def set_ref(self, ref):
        self.call("mace_set_ref", N.ptr(None if ref is None else N.f32(ref)))

    def iterate(self, iters, iter0, rho, use_g, tol, n_total, with_ref, device_denoise=False) -> float:
        """`iters` MACE iterations on the device; use_g: PnP (v from g).  device_denoise: apply the
        loaded K5 denoiser g = H(wbar) inside the loop after every iteration."""
        ms = ctypes.c_float(0.0)
        mode = 2 if (use_g and device_denoise) else int(bool(use_g))
        self.call("mace_iterate", int(iters), int(iter0), float(rho), mode, float(tol), int(n_total),
                  int(bool(with_ref)), ctypes.byref(ms))
        return float(ms.value)

    def k2_timing(self, enable: bool):
        ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
        self.call("mace_k2_timing", int(bool(enable)), ctypes.byref(ms), ctypes.byref(n))
        return ms.value, n.value

    # ---- consensus over NVLink peer memory (k_peer.cuh)
    def peer_bytes(self, world) -> int:
        b = ctypes.c_size_t(0)
        self.call("mace_peer_bytes", int(world), ctypes.byref(b))
        return int(b.value)

    def peer_setup(self, world, rank, ptrs):
        ptrs = np.ascontiguousarray(ptrs, np.uint64)
        self.call("mace_peer_setup", int(world), int(rank), N.ptr(ptrs))

    def peer_mean(self, n_total):
        self.call("mace_peer_mean", int(n_total))

    def iterate_peer(self, iters, iter0, rho, use_g, tol, n_total, device_denoise=False) -> float:
        ms = ctypes.c_float(0.0)
        mode = 2 if (use_g and device_denoise) else int(bool(use_g))
        self.call("mace_iterate_peer", int(iters), int(iter0), float(rho), mode, float(tol), int(n_total),
                  ctypes.byref(ms))
        return float(ms.value)

    def iterate_local(self, rho, use_g):
        self.call("mace_iterate_local", float(rho), int(bool(use_g)))

    def iterate_finish(self, n_total, tol, it):
        """after the all-reduce of comm_arrays() on torch_stream() (stream-ordered, no host sync)"""
        self.call("mace_iterate_finish", int(n_total), float(tol), int(it))

    def set_iter(self, it):
        """device iteration counter for iterate_finish(..., it=-1) (graph-captured loops)"""
        self.call("mace_set_iter", int(it))

    def reserve_log(self, n):
        self.call("mace_reserve_log", int(n))

    def add_passes(self, k) -> int:
        out = ctypes.c_int64(0)
        self.call("mace_passes", int(k), ctypes.byref(out))
        return out.value

    def read_log(self, n):
        lg = np.zeros((max(n, 1), 4), np.float64)
        done = np.zeros(2, np.int32)
        self.call("mace_read_log", int(n), N.ptr(lg), N.ptr(done))
        return lg[:n], (int(done[0]), int(done[1]))

    def get_image(self, which, pinned=False) -> np.ndarray:
        """wbar (which=0) or G_H(w) (which=1): shape (n,), or (n_slices, n) for a batch.  pinned: a
        view of the plan's pinned result buffer (overwritten by the next pinned read)."""
        shape = (self.n_slices, self.n) if self.n_slices > 1 else (self.n,)
        out = self._pinned_out(int(np.prod(shape))).reshape(shape) if pinned else np.empty(shape, np.float32)
        self.call("mace_get_image", int(which), N.ptr(out))
        return out

    def set_image(self, which, img):
        img = N.f32(img)
        if img.size != self.n * self.n_slices:
            raise ValueError("image size mismatch")
        self.call("mace_set_image", int(which), N.ptr(img))

    def get_stack(self, pinned=False) -> np.ndarray:
        """(n_local, n) for one slice, (n_slices, n_agents, n) for a batch (pinned: as get_image)."""
        shape = (self.n_slices, self.n_agents, self.n) if self.n_slices > 1 else (self.n_local, self.n)
        out = self._pinned_out(int(np.prod(shape))).reshape(shape) if pinned else np.empty(shape, np.float32)
        self.call("mace_get_stack", N.ptr(out))
        return out


def _convert_into(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (float64 -> float32 into pinned staging) with torch's multi-threaded CPU copy."""
    if src.size < (1 << 16) or src.dtype.kind != "f":
        np.copyto(dst, src, casting="same_kind")
        return
    import torch

    torch.from_numpy(dst).copy_(torch.from_numpy(np.ascontiguousarray(src)))


class _DevArray:
    """Minimal __cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def plan_for(matrices, agent_views, schedule="sv", sv=DEFAULT_SV, colours=DEFAULT_COLOURS, device=0,
             n_slices=1) -> AgentPlan:
    key = ("plan", id(matrices), tuple(tuple(v) for v in agent_views), schedule, sv, colours, device, n_slices)
    return _cached(key, lambda: AgentPlan(matrices, agent_views, schedule, sv, colours, device, n_slices), matrices)
