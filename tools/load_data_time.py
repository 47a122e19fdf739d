"""Time one data load (H2D of y/lambda, k_gather_data, k_sv_consts) of a config's plan on cuda:0.

python tools/load_data_time.py [config]  -> ms per load_data (device-synchronised wall time and the
CUDA-event time on the plan's stream).
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_09278_b200 as mb  # noqa: E402
from paper_1911_09278_b200 import gen  # noqa: E402
from paper_1911_09278_b200.engine import plan_for  # noqa: E402


def plan_stream(plan):
    import ctypes

    s = ctypes.c_void_p()
    plan.call("mace_ctx_stream", ctypes.byref(s))
    return s.value


config = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = gen.CONFIGS[config]
geom, mats, _, y, lam = gen.make_scan(config)
subsets = mb.partition_views(geom.n_views, cfg["n_agents"])
plan = plan_for(mats, [s.view_indices for s in subsets], schedule="sv", sv=8, device=0)
stream = torch.cuda.ExternalStream(plan_stream(plan), device="cuda:0")
for _ in range(3):
    plan.load_data(y, lam)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(stream)
for _ in range(reps):
    plan.load_data(y, lam)
e1.record(stream)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
print(f"config {config}: load_data {wall:.3f} ms wall, {e0.elapsed_time(e1) / reps:.3f} ms on the stream, "
      f"weighted={plan.info().get('weighted')}")
