"""ctypes binding of libmace_b200.so (include/mace_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of any compute entry point raises.  The library is built in-tree by
``__graft_entry__.build()`` (or ``python -m paper_1911_09278_b200._build``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from ._build import LIB

_lib = None
_lock = threading.Lock()

c_int, c_int64, c_double, c_float, c_void_p, c_size_t = (
    ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t)
P = c_void_p

_SIGS = {
    "mace_last_error": (ctypes.c_char_p, []),
    "mace_abi_version": (c_int, []),
    "mace_sysmat_trace": (c_int, [c_int, c_double, c_int, c_int, P, P, P, P, P, c_int, ctypes.POINTER(c_void_p)]),
    "mace_sysmat_view_nnz": (c_int64, [P, c_int]),
    "mace_sysmat_read": (c_int, [ctypes.c_char_p, P, ctypes.POINTER(c_void_p)]),
    "mace_sysmat_take_view": (c_int, [P, c_int, P, P, P]),
    "mace_sysmat_free": (None, [P]),
    "mace_ctx_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "mace_ctx_destroy": (None, [P]),
    "mace_ctx_stream": (c_int, [P, ctypes.POINTER(c_void_p)]),
    "mace_sync": (c_int, [P]),
    "mace_ctx_info": (c_int, [P, P]),
    "mace_agent_info": (c_int, [P, c_int, P]),
    "mace_load_matrix": (c_int, [P, c_int, c_int, c_int, P, P, P]),
    "mace_set_prior": (c_int, [P, c_int, c_double, c_double, c_double, c_double, c_double]),
    "mace_setup_agents": (c_int, [P, c_int, P, P, c_int, c_int, c_int, c_int, c_int]),
    "mace_set_schedule": (c_int, [P, c_double, c_int64]),
    "mace_set_agent_groups": (c_int, [P, c_int]),
    "mace_set_deterministic": (c_int, [P, c_int]),
    "mace_stage_wait": (c_int, [P]),
    "mace_get_batch_consts": (c_int, [P, c_int, P, P]),
    "mace_set_iter": (c_int, [P, c_int]),
    "mace_reserve_log": (c_int, [P, c_int]),
    "mace_passes": (c_int, [P, c_int64, P]),
    "mace_prox_all": (c_int, [P, P, P, c_int, c_double, P, P]),
    "mace_set_agent_params": (c_int, [P, c_int, c_double, c_double, c_int]),
    "mace_load_data": (c_int, [P, P, P]),
    "mace_set_weighting": (c_int, [P, c_int]),
    "mace_set_state": (c_int, [P, c_int, P]),
    "mace_get_state": (c_int, [P, c_int, P]),
    "mace_get_error": (c_int, [P, c_int, P]),
    "mace_get_theta2": (c_int, [P, c_int, P]),
    "mace_refresh": (c_int, [P, c_int]),
    "mace_pass": (c_int, [P, c_int, P, c_int, c_int64, c_int64, P]),
    "mace_forward_project": (c_int, [P, P, P]),
    "mace_cost": (c_int, [P, P, c_double, P, P]),
    "mace_gradient": (c_int, [P, P, c_double, P, P]),
    "mace_back_project": (c_int, [P, P, P]),
    "mace_peer_bytes": (c_int, [P, c_int, P]),
    "mace_peer_setup": (c_int, [P, c_int, c_int, P]),
    "mace_peer_mean": (c_int, [P, c_int]),
    "mace_iterate_peer": (c_int, [P, c_int, c_int, c_double, c_int, c_double, c_int, P]),
    "mace_stack_init": (c_int, [P, P, c_int]),
    "mace_set_ref": (c_int, [P, P]),
    "mace_states_from": (c_int, [P, c_int]),
    "mace_get_image": (c_int, [P, c_int, P]),
    "mace_set_image": (c_int, [P, c_int, P]),
    "mace_get_stack": (c_int, [P, P]),
    "mace_iterate": (c_int, [P, c_int, c_int, c_double, c_int, c_double, c_int, c_int, P]),
    "mace_iterate_local": (c_int, [P, c_double, c_int]),
    "mace_comm_buffers": (c_int, [P, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]),
    "mace_local_sum": (c_int, [P]),
    "mace_mean_from_sum": (c_int, [P, c_int]),
    "mace_iterate_finish": (c_int, [P, c_int, c_double, c_int]),
    "mace_read_log": (c_int, [P, c_int, P, P]),
    "mace_k2_timing": (c_int, [P, c_int, P, P]),
    "mace_cnn_set_weights": (c_int, [P, P, c_int, c_int]),
    "mace_cnn_apply": (c_int, [P]),
    "mace_cnn_run": (c_int, [P, P, P, c_int, c_int, P]),
    "mace_cnn_layer": (c_int, [P, c_int, P, P, c_int, c_int]),
    "mace_sweep_f64": (c_int, [P] * 10 + [c_double, c_double, c_double, c_int, c_double, c_double, c_double,
                                          c_double, c_int, c_int64, c_int64, c_int64, c_int64, P]),
    "mace_agent_csc": (c_int, [c_int, c_int, c_int, P, P, P, c_int, P, P, P, P]),
    "mace_sv_layout_probe": (c_int, [c_int, c_int, c_int, P, P, P, c_int, P, c_int, P, P, P, P]),
    "mace_host_alloc": (c_int, [c_size_t, ctypes.POINTER(c_void_p)]),
    "mace_host_free": (None, [P]),
}


class NativeError(RuntimeError):
    pass


def lib():
    """Load libmace_b200.so (raising if it is absent — never falls back to CPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB):
                raise NativeError(
                    f"{LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().mace_last_error().decode(errors="replace")
        raise NativeError(f"{what}: {msg}" if what else msg)


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(c_void_p)


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)
