"""On-disk formats against files written by the reference's own writers
(tests/golden/make_format_fixtures.py): MACEMAT1 (native reader, vectorised writer), MACESINO1,
MACEIMG1, PGM.  Host-only (no GPU)."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import fileio
from paper_1911_09278_b200.geometry import load_system_matrix, save_system_matrix

G = os.path.join(os.path.dirname(__file__), "golden")


def _fx(name):
    return os.path.join(G, name)


def test_macemat_reader_matches_tracer_in_float32():
    mats = load_system_matrix(_fx("fmt_small.macemat"))
    ref = mb.build_system_matrix(mb.Geometry(12, 1.0, 10, 17, 0.9))
    assert len(mats) == 10
    for a, b in zip(mats, ref):
        assert a.n_channels == 17 and a.n_pixels == 144
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.cols, b.cols)
        assert a.lens.dtype == np.float64
        assert np.array_equal(a.lens, b.lens.astype(np.float32).astype(np.float64))


def test_macemat_writer_is_byte_identical(tmp_path):
    mats = mb.build_system_matrix(mb.Geometry(12, 1.0, 10, 17, 0.9))
    out = tmp_path / "m.macemat"
    save_system_matrix(out, mats)
    assert out.read_bytes() == open(_fx("fmt_small.macemat"), "rb").read()
    back = load_system_matrix(out)
    assert all(np.array_equal(a.cols, b.cols) for a, b in zip(back, mats))


def test_sinogram_and_image_round_trip_byte_identical(tmp_path):
    src = np.load(_fx("fmt_small_src.npz"))
    y, w = fileio.load_sinogram(_fx("fmt_small.macesino"))
    assert np.array_equal(y, src["y"].astype(np.float32).astype(np.float64))
    assert np.array_equal(w, src["w"].astype(np.float32).astype(np.float64))
    fileio.save_sinogram(tmp_path / "s", src["y"], src["w"])
    assert (tmp_path / "s").read_bytes() == open(_fx("fmt_small.macesino"), "rb").read()
    img = fileio.load_image(_fx("fmt_small.maceimg"))
    assert img.shape == (12, 12)
    assert np.array_equal(img, src["img"].astype(np.float32).astype(np.float64))
    fileio.save_image(tmp_path / "i", src["img"], 12, 12)
    assert (tmp_path / "i").read_bytes() == open(_fx("fmt_small.maceimg"), "rb").read()
    fileio.save_pgm(tmp_path / "p.pgm", src["img"])
    assert (tmp_path / "p.pgm").read_bytes() == open(_fx("fmt_small.pgm"), "rb").read()


def test_bad_magic_and_truncation_raise(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTMACE\n1 1 1\n")
    with pytest.raises(ValueError):
        load_system_matrix(bad)
    with pytest.raises(ValueError):
        fileio.load_image(bad)
    with pytest.raises(ValueError):
        fileio.load_sinogram(bad)
    data = open(_fx("fmt_small.macemat"), "rb").read()
    trunc = tmp_path / "t.macemat"
    trunc.write_bytes(data[: len(data) // 2])
    with pytest.raises(ValueError):
        load_system_matrix(trunc)
    with pytest.raises(OSError):
        load_system_matrix(tmp_path / "missing.macemat")


def test_roi_mask_matches_definition():
    geom = mb.Geometry(13, 0.7, 4, 5, 0.7)
    m = mb.roi_mask(geom)
    half = 0.5 * geom.image_width
    c = (np.arange(13) + 0.5) * 0.7 - half
    xx, yy = np.meshgrid(c, c)
    assert np.array_equal(m, ((xx ** 2 + yy ** 2) <= half ** 2).ravel())
