"""Writes small on-disk format fixtures with the REFERENCE's own writers (run in the build
container, where /root/reference exists; the outputs are committed):

    tests/golden/fmt_small.macemat   save_system_matrix (geometry.py:293-313), 12x12, 10 views x 17 ch
    tests/golden/fmt_small.macesino  save_sinogram (fileio.py:47-60)
    tests/golden/fmt_small.maceimg   save_image (fileio.py:25-32)
    tests/golden/fmt_small.pgm       save_pgm (fileio.py:75-)

    python tests/golden/make_format_fixtures.py
"""
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/tmp/refpkg_fmt"
if not os.path.exists(SRC):
    shutil.copytree("/root/reference/pkg", SRC)
sys.path.insert(0, os.path.join(SRC, "src"))
from macetomo import fileio, geometry  # noqa: E402

geom = geometry.Geometry(12, 1.0, 10, 17, 0.9)
mats = geometry.build_system_matrix(geom)
geometry.save_system_matrix(os.path.join(HERE, "fmt_small.macemat"), mats)
rng = np.random.default_rng(5)
y = rng.random((10, 17)) * 3.0
w = rng.integers(1, 1000, (10, 17)).astype(np.float64)
fileio.save_sinogram(os.path.join(HERE, "fmt_small.macesino"), y, w)
img = rng.random((12, 12)) * 0.02 - 0.005
fileio.save_image(os.path.join(HERE, "fmt_small.maceimg"), img, 12, 12)
fileio.save_pgm(os.path.join(HERE, "fmt_small.pgm"), img)
np.savez(os.path.join(HERE, "fmt_small_src.npz"), y=y, w=w, img=img)
print("wrote fixtures")
