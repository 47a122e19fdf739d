"""Timeline of the persistent K5 kernel (k_conv64_seq) from a K5SEQ_TRACE build:
    MACE_LIB=/tmp/libk5t.so MACE_NVCC_EXTRA=-DK5SEQ_TRACE python -c "from paper_1911_09278_b200 import _build; _build.build(force=True)"
    MACE_LIB=/tmp/libk5t.so MACE_K5_SEQ=1 python tools/k5seq_trace.py
Per layer (median over CTAs, microseconds from the kernel's first stamp): weights-free seen,
neighbour flags passed, weights landed, first unit issued, last unit issued, layer published."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_09278_b200 import _native as N  # noqa: E402
from paper_1911_09278_b200.denoisers import CnnDenoiser, cnn_weights  # noqa: E402

n = 512
H = CnnDenoiser(n, weights=cnn_weights(0, scale=1.0))
x = np.random.default_rng(0).random(n * n)
for _ in range(3):
    H(x)
print("last ms", H.last_ms)
L = N.lib()
buf = np.zeros((148, 16, 6), np.uint64)
f = getattr(L, "mace_k5seq_trace")
f.argtypes = [ctypes.c_void_p]
assert f(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf.astype(np.float64)
ncta = int((t[:, 0, 1] > 0).sum())
t = t[:ncta]
t0 = t[:, 0, 1].min()
rel = (t - t0) / 1e3
names = ["wfree", "flags", "weights", "unit0", "unitN", "publish"]
print("layer " + " ".join(f"{k:>9s}" for k in names) + "   (median us; spread of publish = max-min)")
for l in range(15):
    row = rel[:, l, :]
    med = np.median(row, axis=0)
    spread = row[:, 5].max() - row[:, 5].min()
    print(f"{l:5d} " + " ".join(f"{v:9.2f}" for v in med) + f"   {spread:6.2f}")
