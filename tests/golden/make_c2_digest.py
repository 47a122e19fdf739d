"""Config-2 system-matrix digest from the reference itself (build container only).

The reference's build_system_matrix holds every view in one list (23 GB at config 2);
this script runs the same per-view loop body with the reference's own _trace_ray and
Geometry (geometry.py:228-258), views traced in a process pool and hashed in view
order with make_golden.mat_digest's recipe, and adds "c2" to sysmat_digests.json.

    python tests/golden/make_c2_digest.py     # ~1 min on 8 cores
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

PARAMS = (1024, 0.125, 1440, 1450, 0.125)
_mt = None


def _views(args):
    k0, k1 = args
    import macetomo.geometry as geo
    geom = geo.Geometry(*PARAMS)
    offsets = geom.channel_offsets()
    out = []
    for k in range(k0, k1):  # geometry.py:236-256
        theta = geom.view_angles[k]
        ux, uy = -np.sin(theta), np.cos(theta)
        ex, ey = np.cos(theta), np.sin(theta)
        row_ptr = np.zeros(geom.n_channels + 1, dtype=np.int64)
        cols, lens = [], []
        for d in range(geom.n_channels):
            s = offsets[d]
            pix, seg = geo._trace_ray(s * ex, s * ey, ux, uy, geom)
            row_ptr[d + 1] = row_ptr[d] + pix.shape[0]
            cols.append(pix)
            lens.append(seg)
        out.append((row_ptr, np.concatenate(cols), np.concatenate(lens)))
    return out


def main():
    global _mt
    _mt = import_reference()
    import macetomo.geometry  # noqa: F401
    h = hashlib.sha256()
    nnz = 0
    jobs = [(k, min(k + 8, PARAMS[2])) for k in range(0, PARAMS[2], 8)]
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for part in pool.imap(_views, jobs):
            for rp, cols, lens in part:
                h.update(np.ascontiguousarray(rp, np.int64).tobytes())
                h.update(np.ascontiguousarray(cols, np.int32).tobytes())
                h.update(np.ascontiguousarray(lens, np.float64).tobytes())
                nnz += int(rp[-1])
    path = os.path.join(HERE, "sysmat_digests.json")
    d = json.load(open(path))
    d["c2"] = {"params": list(PARAMS), "sha256": h.hexdigest(), "nnz": nnz,
               "how": "reference geometry._trace_ray per view (make_c2_digest.py)"}
    json.dump(d, open(path, "w"), indent=1)
    print("c2", d["c2"])


if __name__ == "__main__":
    main()
