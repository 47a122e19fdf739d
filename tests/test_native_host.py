"""CPU tests of libmace_b200.so: exports, the native tracer (bit-exact to the
reference), the agent stacking (bit-exact to the reference's CSC) and the
super-voxel layout (a lossless re-packing).  No GPU calls."""

from __future__ import annotations

import hashlib
import json
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, ROOT, small_problem, unpack_views
from golden.make_golden import GEOMS

from paper_1911_09278_b200 import _native as N
from paper_1911_09278_b200.geometry import Geometry, build_system_matrix, global_csr, partition_views


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "mace_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mace_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    syms = _header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert L.mace_abi_version() == 1


@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_native_tracer_bit_exact_vs_reference_golden(golden, gi):
    ns, pp, nv, nc, cp = GEOMS[gi]
    mats = build_system_matrix(Geometry(ns, pp, nv, nc, cp))
    ref = unpack_views(golden, f"geom{gi}", nv, nc, ns * ns)
    for m, r in zip(mats, ref):
        assert np.array_equal(m.row_ptr, r.row_ptr)
        assert m.cols.dtype == np.int32 and np.array_equal(m.cols, r.cols)
        assert np.array_equal(m.lens.view(np.uint64), r.lens.view(np.uint64))


@pytest.mark.parametrize("seed", range(6))
def test_native_tracer_bit_exact_vs_oracle_random_geometry(seed):
    rng = np.random.default_rng(seed)
    ns = int(rng.integers(2, 40))
    nv = int(rng.integers(1, 50))
    nc = int(rng.integers(1, 70))
    pp = float(rng.uniform(0.1, 3.0))
    cp = float(rng.uniform(0.1, 3.0))
    mats = build_system_matrix(Geometry(ns, pp, nv, nc, cp))
    ref = O.build_system_matrix(ns, pp, nv, nc, cp)
    for m, r in zip(mats, ref):
        assert np.array_equal(m.row_ptr, r.row_ptr)
        assert np.array_equal(m.cols, r.cols)
        assert np.array_equal(m.lens.view(np.uint64), r.lens.view(np.uint64))


def _digest(mats):
    h = hashlib.sha256()
    for m in mats:
        h.update(np.ascontiguousarray(m.row_ptr, np.int64).tobytes())
        h.update(np.ascontiguousarray(m.cols, np.int32).tobytes())
        h.update(np.ascontiguousarray(m.lens, np.float64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_native_tracer_full_config_digest(name):
    """Bit-exact at the benchmark sizes: SHA-256 of the reference's own output (make_golden.py --hashes)."""
    d = json.load(open(os.path.join(GOLDEN, "sysmat_digests.json")))[name]
    ns, pp, nv, nc, cp = d["params"]
    mats = build_system_matrix(Geometry(int(ns), pp, int(nv), int(nc), cp))
    assert sum(m.nnz for m in mats) == d["nnz"]
    assert _digest(mats) == d["sha256"]


CASES = ["pq", "pg", "pg2", "pq2", "pg3"]


@pytest.mark.parametrize("name", CASES)
def test_agent_stacking_bit_exact_vs_reference(golden, name):
    seed, ns, nv, nc, beta, sx, Nsub, agent, sigma, _ = golden[f"{name}_meta"]
    ns, nv, nc, Nsub, agent = int(ns), int(nv), int(nc), int(Nsub), int(agent)
    mats = build_system_matrix(Geometry(ns, 1.0, nv, nc, ns / nc * 1.1))
    rp, cols, vals = global_csr(mats)
    views = np.array(partition_views(nv, Nsub)[agent].view_indices, np.int32)
    n = ns * ns
    col_ptr = np.zeros(n + 1, np.int64)
    N.check(N.lib().mace_agent_csc(ns, nc, nv, N.ptr(rp), N.ptr(cols), N.ptr(vals), len(views), N.ptr(views),
                                   N.ptr(col_ptr), None, None))
    rows = np.zeros(col_ptr[-1], np.uint32)
    v32 = np.zeros(col_ptr[-1], np.float32)
    N.check(N.lib().mace_agent_csc(ns, nc, nv, N.ptr(rp), N.ptr(cols), N.ptr(vals), len(views), N.ptr(views),
                                   N.ptr(col_ptr), N.ptr(rows), N.ptr(v32)))
    assert np.array_equal(col_ptr, golden[f"{name}_colptr"])
    assert np.array_equal(rows.astype(np.int64), golden[f"{name}_rowidx"])
    assert np.array_equal(v32, golden[f"{name}_aval"].astype(np.float32))


def _sv_probe(mats, views, svs):
    ns = int(np.sqrt(mats[0].n_pixels))
    nc = mats[0].n_channels
    rp, cols, vals = global_csr(mats)
    views = np.asarray(views, np.int32)
    stats = np.zeros(6, np.int64)
    L = N.lib()
    N.check(L.mace_sv_layout_probe(ns, nc, len(mats), N.ptr(rp), N.ptr(cols), N.ptr(vals), len(views),
                                   N.ptr(views), svs, N.ptr(stats), None, None, None))
    k = int(stats[5])
    pix, row, val = np.zeros(k, np.int32), np.zeros(k, np.int32), np.zeros(k, np.float32)
    N.check(L.mace_sv_layout_probe(ns, nc, len(mats), N.ptr(rp), N.ptr(cols), N.ptr(vals), len(views),
                                   N.ptr(views), svs, N.ptr(stats), N.ptr(pix), N.ptr(row), N.ptr(val)))
    return stats, pix, row, val


@pytest.mark.parametrize("ns,nv,nc,Nsub,svs", [(6, 12, 9, 3, 2), (13, 17, 23, 4, 4), (32, 45, 47, 4, 8),
                                                (20, 30, 31, 1, 6), (9, 8, 11, 2, 16)])
def test_sv_layout_is_lossless_repacking(ns, nv, nc, Nsub, svs):
    mats = build_system_matrix(Geometry(ns, 1.0, nv, nc, 1.0))
    ref = O.build_system_matrix(ns, 1.0, nv, nc, 1.0)
    for a, sub in enumerate(O.partition_views(nv, Nsub)):
        stats, pix, row, val = _sv_probe(mats, sub, svs)
        ag = O.Agent(ref, np.zeros((nv, nc)), np.ones((nv, nc)), sub, Nsub, 1.0, O.Prior(), ns)
        csc_pix = np.repeat(np.arange(ns * ns), np.diff(ag.col_ptr))
        want = sorted(zip(csc_pix.tolist(), ag.row_idx.tolist(), ag.a_val.astype(np.float32).tolist()))
        got = sorted(zip(pix.tolist(), row.tolist(), val.tolist()))
        assert stats[4] == 0  # no duplicate (row, pixel) entries in the reference matrices
        assert got == want
        assert stats[0] % 64 == 0 and 0 < stats[1] <= 255  # lane slots; widest band window


def test_bad_views_rejected():
    mats = build_system_matrix(Geometry(4, 1.0, 2, 3, 1.0))
    rp, cols, vals = global_csr(mats)
    views = np.array([0, 5], np.int32)
    col_ptr = np.zeros(17, np.int64)
    rc = N.lib().mace_agent_csc(4, 3, 2, N.ptr(rp), N.ptr(cols), N.ptr(vals), 2, N.ptr(views), N.ptr(col_ptr),
                                None, None)
    assert rc != 0 and b"out of range" in N.lib().mace_last_error()
