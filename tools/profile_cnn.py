"""Driver for K5 timing / ncu: H(x) on an n x n image, `reps` times after a warm-up."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_09278_b200.denoisers import CnnDenoiser, cnn_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
H = CnnDenoiser(a.n, weights=cnn_weights(0, scale=1.0))
x = np.random.default_rng(0).random(a.n * a.n)
H(x)
ts = []
for _ in range(a.reps):
    H(x)
    ts.append(H.last_ms)
flop = 2.0 * a.n * a.n * (15 * 64 * 64 * 9 + 2 * 64 * 9)
print(f"K5 {a.n}^2: {min(ts):.3f} ms best of {a.reps} -> {flop / (min(ts) * 1e-3) / 1e12:.1f} TFLOP/s")
