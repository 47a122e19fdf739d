"""2D parallel-beam geometry, view subsets and the system matrix.

Mirrors the reference's public types and functions
(/root/reference/pkg/src/macetomo/geometry.py) so that a ``ReconProblem``
built for either package works with both.  ``build_system_matrix`` runs the
native tracer (csrc/sysmat.cpp, bit-exact to geometry.py:177-258) on all host
cores; ``forward_project`` runs kernel K3 on the GPU.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

__all__ = [
    "Geometry",
    "SparseViewMatrix",
    "ViewSubset",
    "partition_views",
    "build_system_matrix",
    "forward_project",
    "global_csr",
    "save_system_matrix",
    "load_system_matrix",
    "back_project",
    "roi_mask",
    "MATRIX_MAGIC",
]

MATRIX_MAGIC = "MACEMAT1"


@dataclass(frozen=True)
class Geometry:
    """Scan geometry (geometry.py:39-101): n_side^2 pixels of side pixel_pitch
    centred on the origin, row 0 at the top; n_views angles in [0, pi); view k
    has n_channels parallel rays offset by (d - (n_channels-1)/2) * channel_pitch."""

    n_side: int
    pixel_pitch: float
    n_views: int
    n_channels: int
    channel_pitch: float
    view_angles: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        for name in ("n_side", "n_views", "n_channels"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.pixel_pitch <= 0 or self.channel_pitch <= 0:
            raise ValueError("pitches must be > 0")
        if self.view_angles is None:
            ang = np.arange(self.n_views) * (np.pi / self.n_views)
        else:
            ang = np.asarray(self.view_angles, dtype=np.float64)
            if ang.shape != (self.n_views,):
                raise ValueError("view_angles must have length n_views")
            if np.any(ang < 0.0) or np.any(ang >= np.pi):
                raise ValueError("view_angles must lie in [0, pi)")
            if self.n_views > 1 and np.any(np.diff(ang) <= 0.0):
                raise ValueError("view_angles must be strictly increasing")
        ang = np.ascontiguousarray(ang, dtype=np.float64)
        ang.setflags(write=False)
        object.__setattr__(self, "view_angles", ang)

    @property
    def n_pixels(self) -> int:
        return self.n_side * self.n_side

    @property
    def image_width(self) -> float:
        return self.n_side * self.pixel_pitch

    def channel_offsets(self) -> np.ndarray:
        d = np.arange(self.n_channels, dtype=np.float64)
        return (d - (self.n_channels - 1) / 2.0) * self.channel_pitch


@dataclass(frozen=True)
class ViewSubset:
    """Views owned by one agent (geometry.py:104-112)."""

    subset_index: int
    view_indices: tuple

    def __len__(self) -> int:
        return len(self.view_indices)


@dataclass
class SparseViewMatrix:
    """One view's CSR operator: row d (channel) owns cols/lens[row_ptr[d]:row_ptr[d+1]]
    (geometry.py:115-158).  cols int32 sorted per row, lens float64."""

    view_index: int
    n_channels: int
    n_pixels: int
    row_ptr: np.ndarray
    cols: np.ndarray
    lens: np.ndarray

    def __post_init__(self):
        if self.row_ptr.shape != (self.n_channels + 1,):
            raise ValueError("row_ptr must have length n_channels + 1")
        if self.cols.shape != self.lens.shape:
            raise ValueError("cols and lens must have equal length")

    @property
    def nnz(self) -> int:
        return int(self.cols.shape[0])

    def row(self, d: int):
        lo, hi = self.row_ptr[d], self.row_ptr[d + 1]
        return self.cols[lo:hi], self.lens[lo:hi]


def partition_views(n_views: int, n_subsets: int) -> list[ViewSubset]:
    """Interleaved subsets {m : m mod N == i} (geometry.py:161-174)."""
    if n_subsets < 1:
        raise ValueError("n_subsets must be >= 1")
    if n_subsets > n_views:
        raise ValueError("n_subsets must not exceed n_views")
    return [ViewSubset(i, tuple(range(i, n_views, n_subsets))) for i in range(n_subsets)]


def build_system_matrix(geom: Geometry, n_threads: int = 0) -> list[SparseViewMatrix]:
    """Trace every ray with the native tracer; output identical (bitwise) to the reference's."""
    L = N.lib()
    ang = geom.view_angles
    ux = np.ascontiguousarray(-np.sin(ang))  # computed in numpy, as geometry.py:237-239 does
    uy = np.ascontiguousarray(np.cos(ang))
    ex = np.ascontiguousarray(np.cos(ang))
    ey = np.ascontiguousarray(np.sin(ang))
    offs = np.ascontiguousarray(geom.channel_offsets())
    h = ctypes.c_void_p()
    N.check(L.mace_sysmat_trace(geom.n_side, float(geom.pixel_pitch), geom.n_views, geom.n_channels, N.ptr(ux),
                                N.ptr(uy), N.ptr(ex), N.ptr(ey), N.ptr(offs), int(n_threads), ctypes.byref(h)),
            "sysmat_trace")
    out = []
    try:
        for k in range(geom.n_views):
            nnz = L.mace_sysmat_view_nnz(h, k)
            rp = np.empty(geom.n_channels + 1, np.int64)
            cols = np.empty(nnz, np.int32)
            lens = np.empty(nnz, np.float64)
            N.check(L.mace_sysmat_take_view(h, k, N.ptr(rp), N.ptr(cols), N.ptr(lens)), "sysmat_take_view")
            out.append(SparseViewMatrix(k, geom.n_channels, geom.n_pixels, rp, cols, lens))
    finally:
        L.mace_sysmat_free(h)
    return out


def back_project(matrices, sinogram, device: int = 0) -> np.ndarray:
    """Exact transpose of forward_project (geometry.py:273-282) on the GPU, fp64 accumulation
    (float32 operands, like forward_project)."""
    from .engine import operator_for

    sinogram = np.asarray(sinogram, dtype=np.float64)
    expected = (len(matrices), matrices[0].n_channels)
    if sinogram.shape != expected:
        raise ValueError(f"sinogram must have shape {expected}, got {sinogram.shape}")
    return operator_for(matrices, device=device).back_project(sinogram)


def roi_mask(geom: Geometry) -> np.ndarray:
    """Pixels whose centres fall in the inscribed circle (geometry.py:285-290)."""
    half = 0.5 * geom.image_width
    c = (np.arange(geom.n_side) + 0.5) * geom.pixel_pitch - half
    xx, yy = np.meshgrid(c, c)
    return ((xx**2 + yy**2) <= half**2).ravel()


def _take_views(L, h, n_views, n_channels, n_pixels) -> list[SparseViewMatrix]:
    out = []
    for k in range(n_views):
        nnz = L.mace_sysmat_view_nnz(h, k)
        rp = np.empty(n_channels + 1, np.int64)
        cols = np.empty(nnz, np.int32)
        lens = np.empty(nnz, np.float64)
        N.check(L.mace_sysmat_take_view(h, k, N.ptr(rp), N.ptr(cols), N.ptr(lens)), "sysmat_take_view")
        out.append(SparseViewMatrix(k, n_channels, n_pixels, rp, cols, lens))
    return out


def save_system_matrix(path, matrices: list[SparseViewMatrix]) -> None:
    """Write the MACEMAT1 cache (geometry.py:293-313): ASCII magic line, ASCII "n_views n_channels n",
    then per view, per row a uint32 LE count and (uint32 LE pixel, float32 LE length) pairs.  One
    vectorised record block per view (byte-identical to the reference's per-row writer)."""
    with open(path, "wb") as fh:
        fh.write(f"{MATRIX_MAGIC}\n".encode("ascii"))
        fh.write(f"{len(matrices)} {matrices[0].n_channels} {matrices[0].n_pixels}\n".encode("ascii"))
        for mat in matrices:
            rp = np.asarray(mat.row_ptr, np.int64)
            counts = np.diff(rp).astype("<u4")
            nnz = int(rp[-1] - rp[0])
            words = np.empty(mat.n_channels + 2 * nnz, "<u4")
            # word position of row d's count: d + 2 * (entries before row d)
            pos = np.arange(mat.n_channels) + 2 * (rp[:-1] - rp[0])
            words[pos] = counts
            entry_row = np.repeat(np.arange(mat.n_channels), counts)
            epos = entry_row + 1 + 2 * np.arange(nnz)
            words[epos] = np.asarray(mat.cols[rp[0]:rp[-1]], "<u4")
            words[epos + 1] = np.asarray(mat.lens[rp[0]:rp[-1]], "<f4").view("<u4")
            fh.write(words.tobytes())


def load_system_matrix(path) -> list[SparseViewMatrix]:
    """Read a MACEMAT1 file (geometry.py:316-342; float32 lengths returned as float64) with the
    native reader: one sequential pass in C++ into the per-view CSR."""
    L = N.lib()
    dims = np.zeros(3, np.int64)
    h = ctypes.c_void_p()
    rc = L.mace_sysmat_read(os.fsencode(path), N.ptr(dims), ctypes.byref(h))
    if rc != 0:
        msg = L.mace_last_error().decode(errors="replace")
        if "cannot open" in msg:
            raise OSError(msg)
        raise ValueError(msg)  # bad magic / header, truncated file, index out of range
    try:
        return _take_views(L, h, int(dims[0]), int(dims[1]), int(dims[2]))
    finally:
        L.mace_sysmat_free(h)


def global_csr(matrices) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Concatenate per-view CSR blocks into one (n_views*n_ch) x n CSR with float32 values."""
    n_ch = matrices[0].n_channels
    nnz = np.fromiter((len(m.cols) for m in matrices), np.int64, len(matrices))
    base = np.concatenate(([0], np.cumsum(nnz)[:-1]))
    rp = np.empty(len(matrices) * n_ch + 1, np.int64)
    for k, m in enumerate(matrices):
        rp[k * n_ch:(k + 1) * n_ch] = np.asarray(m.row_ptr[:-1], np.int64) + base[k]
    rp[-1] = int(nnz.sum())
    cols = np.concatenate([np.asarray(m.cols, np.int32) for m in matrices]) if len(matrices) else np.empty(0, np.int32)
    vals = np.concatenate([np.asarray(m.lens, np.float32) for m in matrices]) if len(matrices) else np.empty(0, np.float32)
    return rp, np.ascontiguousarray(cols), np.ascontiguousarray(vals)


def forward_project(matrices, x, device: int = 0) -> np.ndarray:
    """out[k, d] = sum_j A[k, d, j] x[j] on the GPU (kernel K3; geometry.py:261-270)."""
    from .engine import operator_for

    n = matrices[0].n_pixels
    x = np.asarray(x)
    if x.shape != (n,):
        raise ValueError(f"image must have shape ({n},), got {x.shape}")
    op = operator_for(matrices, device=device)
    return op.forward_project(x).astype(np.float64)
