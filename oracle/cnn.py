"""TEST INFRASTRUCTURE ONLY — CPU oracle for the K5 PnP denoiser (BASELINE config 3).

H(x) = x - net(x), net = 17 bias-free 3x3 convs (1->64, 15x 64->64, 64->1), ReLU between,
zero padding; bf16 weights; activations rounded to bf16 between layers (the GPU kernel's
rounding points), fp32... here fp64 accumulation (torch CPU), so only accumulation-order
rounding separates it from the tensor-core path.  The reference accepts any callable as the
denoiser (mace.py:385-404); this is the callable both sides use.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def bf16_round(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(t.dtype)


def cnn_apply(x, weights, n_side: int) -> np.ndarray:
    """x: flat (n_side*n_side,) image; weights: 17 OIHW float arrays holding bf16 values."""
    xt = torch.from_numpy(np.asarray(x, np.float64).reshape(1, 1, n_side, -1))
    h = bf16_round(xt.to(torch.float32)).to(torch.float64)
    for i, w in enumerate(weights):
        wt = torch.from_numpy(np.asarray(w, np.float64))
        h = F.conv2d(h, wt, padding=1)
        if i < len(weights) - 1:
            h = bf16_round(torch.relu(h).to(torch.float32)).to(torch.float64)
    return (xt - h).reshape(-1).numpy()
