"""Benchmark: MACE voxel-updates/s and time-to-RMSE on BASELINE config 2 (1024^2, 1440 views x
1450 channels, N = 16 view-interleaved agents, rho = 0.8, 50 iterations, qGGMRF) -- the
metric's 1/2/4/8-GPU strong-scaling config -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

``--gpus N`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks (one process per GPU, agent i on rank i mod N).

A step is one full MACE solve of the config's iteration budget on the seeded
synthetic scan (gen.make_scan).  ``value`` = total voxel updates (N agents x n
pixels x iterations x steps, all ranks) / max-over-ranks device time, inputs
resident in HBM.  ``e2e`` = the same metric through the public API
(mace_solve on host numpy arrays: H2D of y / weights, D2H of image + stack
inside the timed region).  The per-iteration record stream (1.9 GB at config 1,
15.6 GB at config 2; ``config.l2``) exceeds the 126 MB L2, so no L2 flush is
needed between steps.

``--impl reference`` times the CPU oracle (oracle/, the restatement of the
reference's numba hot loop, all host threads) on a bounded sample of the same
workload and prints the same metric with "impl": "reference".  That arm never
loads this repo's CUDA library: the scan is traced by the oracle's tracer
(checked against the reference's SHA-256) and the data synthesised by gen.py
loaded as a plain module.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MACE voxel-updates/s"
# fresh-solve iterations run for time-to-RMSE <= 1e-3 (covers the measured first-passage iteration)
TTR_ITERS = {0: 1500, 1: 3000, 2: 8000}
UNIT = "voxel-updates/s"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(gpus: int, argv: list[str]) -> list[str] | None:
    """The torchrun command that runs this script on `gpus` ranks, or None when no re-launch is
    needed (one GPU, or already inside a torchrun environment of the right size)."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != gpus:
            raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
        return None
    if gpus <= 1:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]


def load_gen():
    """paper_1911_09278_b200/gen.py (the workload recipe: phantom, Poisson draw, config table) as a
    plain module, without importing the package (the reference arm must not load libmace_b200)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_bench_gen", os.path.join(ROOT, "paper_1911_09278_b200", "gen.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def l2_mb():
    try:
        import torch

        return round(torch.cuda.get_device_properties(0).L2_cache_size / 2 ** 20)
    except Exception:
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = []
        try:
            for line in open(self.f.name):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def algorithmic_bytes_per_pass(plan, n_agents_local) -> tuple[int, dict]:
    """B_upd = 8 c + 16 + 12 R_i / n per voxel update; per K2 launch that is
    8 nnz (A: f32 value + i32 row) + 16 n N (z r/w, v, theta2) + 12 sum R_i (e r/w, lambda)."""
    nnz = 0
    ent = 0
    R = 0
    for a in range(n_agents_local):
        info = plan.agent_info(a)
        nnz += info["nnz"]
        ent += info["entries"]
        R += info["R"]
    n = plan.n
    alg = 8 * nnz + 16 * n * n_agents_local + 12 * R
    # bytes the lane-per-view super-voxel layout streams per launch (layout.cpp): slot records
    # (ng*32*K lengths + 32 offset words per pixel slot, 4 slots per batch), 64 B of batch constants
    # per batch, the tile's lambda band (ng x wcap x 32 floats; not with weighted records, whose
    # lengths carry sqrt(lambda)) and z/v/w per pixel
    lay_bytes = 0
    ci = plan.info()
    S = ci["S"]
    band = 0 if ci.get("weighted") else 128
    if S < plan.n_side:
        nb = 4 * (((S // 2) ** 2 + 3) // 4)
        for a in range(n_agents_local):
            info = plan.agent_info(a)
            V = len(plan.agent_views[a]) if hasattr(plan, "agent_views") else None
            ng = -(-V // 32) if V else 3
            rec = ng * 64 + 32
            lay_bytes += info["n_sv"] * (nb * (4 * rec * 4 + 64) + ng * info["ctx_wcap"] * band)
        lay_bytes += 16 * n * n_agents_local
    return alg, {"nnz": nnz, "layout_entries": ent, "rows": R, "layout_bytes": lay_bytes,
                 "c_mean": nnz / (n * n_agents_local)}


def k2_traffic(config, sv):
    """dram read + write bytes per K2 launch from the committed ncu --set full captures (profiles/)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_k2_traffic.json")))
    except (OSError, ValueError):
        return None
    e = t.get(str(config))
    return e["dram_bytes_per_launch"] if e and e.get("sv_side") == sv else None


def run_cpu_test(args):
    """Test hook (--cpu-test): the same rank layout and max-over-ranks timing as run_ours, on CPU
    with gloo and the oracle-backed plan of tests/cpu_backend.py, so the --gpus N launch path
    (re-exec under torch.distributed.run, one process per rank) is exercised without a GPU."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import paper_1911_09278_b200 as mb
    from conftest import small_problem
    from cpu_backend import CpuPlan

    _, y, w = small_problem(31, 8, 16, 11)
    geom = mb.Geometry(8, 1.0, 16, 11, 8 / 11 * 1.1)
    prob = mb.ReconProblem(geom, mb.build_system_matrix(geom), y, w, mb.PriorParams("qggmrf", 1.0, sigma_x=0.5))
    cfg = mb.MaceConfig(n_subsets=4, rho=0.8, sigma=0.2, max_outer=12, tol=1e-300, residuals="none")
    res = None
    for _ in range(args.warmup):
        res = _solve_api(mb, prob, cfg, True if world > 1 else None, backend=CpuPlan)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = _solve_api(mb, prob, cfg, True if world > 1 else None, backend=CpuPlan)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    updates = cfg.n_subsets * geom.n_pixels * cfg.max_outer * args.steps
    line = {"metric": METRIC, "value": updates / float(dt), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "cpu_test": True,
            "ranks_agents": {r: [i for i in range(cfg.n_subsets) if i % world == r] for r in range(world)},
            "image_sum": float(np.sum(res.image))}
    if args.ttr_iters > 0:  # the multi-rank time-to-RMSE path against a long solve's image
        import dataclasses

        ref = _solve_api(mb, prob, dataclasses.replace(cfg, max_outer=400), True if world > 1 else None,
                         backend=CpuPlan).image
        line["time_to_rmse_1e-3"] = time_to_rmse_ranks(mb, prob, cfg, True if world > 1 else None, ref,
                                                       args.ttr_iters, float(dt) * 1e3 / (args.steps * cfg.max_outer),
                                                       "400-iteration solve", backend=CpuPlan)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_1911_09278_b200 as mb
    from paper_1911_09278_b200 import gen
    from paper_1911_09278_b200.engine import plan_for

    cfg = gen.CONFIGS[args.config]
    N, iters = cfg["n_agents"], args.iters or cfg["iters"]
    pnp = args.config == 3  # config 3: PnP MACE with the 17-layer CNN denoiser (K5) as the prior agent
    t0 = time.time()
    geom, mats, phantom, y, lam = gen.make_scan(args.config)
    t_scan = time.time() - t0
    prior = mb.PriorParams("qggmrf", beta=cfg["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
    prob = mb.ReconProblem(geom, mats, y, lam, prior)
    mcfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=cfg["sigma"], max_outer=iters, tol=1e-300,
                         residuals="none", schedule=args.schedule, sv_side=args.sv, device=local,
                         **({"mode": "pnp", "denoiser": mb.DenoiserSpec("identity")} if pnp else {}))
    den = mb.denoisers.CnnDenoiser(geom.n_side, seed=0, device=local) if pnp else None
    comm = True if world > 1 else None
    subsets = mb.partition_views(geom.n_views, N)
    local_agents = [i for i in range(N) if i % world == rank]
    t0 = time.time()
    plan = plan_for(mats, [subsets[i].view_indices for i in local_agents], schedule=args.schedule, sv=args.sv,
                    device=local)
    t_plan = time.time() - t0
    n = geom.n_pixels
    stream = torch.cuda.ExternalStream(plan_stream(plan), device=f"cuda:{local}")

    peer = world > 1 and args.comm == "peer"
    if peer:
        pcomm = mb.PeerComm()
        pcomm.attach(plan)
        comm = pcomm  # the e2e solves use the same exchange
        if pnp:
            den._load(plan)

    graph_cache = {}
    graphs = True

    def solve_device():
        """one step with inputs resident: stack init, X0 = average(w0), refresh e, `iters` iterations"""
        plan.stack_init(None, N if world == 1 else 0)
        if peer:
            plan.peer_mean(N)
        elif world > 1:
            plan.local_sum()
            mb.mace._resolve_comm(True).allreduce(*plan.comm_arrays()[:1], stream=plan.torch_stream())
            plan.mean_from_sum(N)
        if pnp:
            den.device_apply(plan)  # g = H(wbar)
        plan.states_from(1 if pnp else 0)
        if world == 1:
            plan.iterate(iters, 0, 0.8, pnp, 1e-300, N, False, device_denoise=pnp)
        elif peer:  # consensus over NVLink peer memory, the whole loop on the device
            plan.iterate_peer(iters, 0, 0.8, pnp, 1e-300, N, device_denoise=pnp)
        else:  # NCCL all-reduce on the library stream; whole blocks of iterations replayed as CUDA graphs
            c = mb.mace._resolve_comm(True)
            G = mb.mace.GRAPH_BLOCK
            k = 0
            if graphs and G > 0:
                plan.reserve_log(iters)
                while k + G <= iters:
                    plan.set_iter(k)
                    if "g" not in graph_cache:
                        graph_cache["g"] = mb.mace._capture_block(plan, c, plan.torch_stream(), G, 0.8, pnp, N,
                                                                  1e-300, den)
                    mb.mace._replay(graph_cache["g"], plan.torch_stream())
                    plan.add_passes(G)
                    k += G
            for k in range(k, iters):
                plan.iterate_local(0.8, pnp)
                c.allreduce(*plan.comm_arrays(), stream=plan.torch_stream())
                plan.iterate_finish(N, 1e-300, k)
                if pnp:
                    den.device_apply(plan)

    # resident inputs
    plan.load_data(y, lam)
    plan.set_prior(prior)
    if pnp:  # agents carry only data terms at sqrt(N) sigma (mace.py:263-265)
        plan.set_agent_params(-1, 0.0, 1.0 / (N * cfg["sigma"] ** 2), False)
    else:
        plan.set_agent_params(-1, prior.beta / N, 1.0 / cfg["sigma"] ** 2, False)

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        solve_device()
    plan.k2_timing(True)
    barrier()
    with ClockSampler(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            solve_device()
        ev1.record(stream)
        barrier()
    k2_ms, k2_launches = plan.k2_timing(False)
    ms = ev0.elapsed_time(ev1)
    if world > 1 and k2_launches < iters * args.steps:  # graph replays carry no K2 events: one timed eager solve
        graphs = False
        plan.k2_timing(True)
        solve_device()
        k2_ms, k2_launches = plan.k2_timing(False)
        graphs = True
    lg, done = plan.read_log(iters)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    updates = N * n * iters * args.steps
    value = updates / (ms / 1e3)

    # ---- end to end through the public API (host numpy in, host numpy out)
    for _ in range(1):
        _solve_api(mb, prob, mcfg, comm, den)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = _solve_api(mb, prob, mcfg, comm, den)
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = updates / e2e_s
    h2d = 2 * geom.n_views * geom.n_channels * 4
    d2h = (n + N * n) * 4

    alg, lay = algorithmic_bytes_per_pass(plan, len(local_agents))
    pk = peaks()
    k2_avg_ms = k2_ms / max(k2_launches, 1)
    achieved = alg / (k2_avg_ms / 1e3) / 1e9
    clocks = clk.summary()
    launches_per_step = 3 + 4 * iters + (iters // 50)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded ellipse phantom, "
        "Poisson counts; gen.make_scan)",
        "config": {"workload": f"BASELINE config {args.config}: {geom.n_side}^2, {geom.n_views} views x "
                   f"{geom.n_channels} ch, N={N} agents, {iters} iterations, rho=0.8, qGGMRF beta={cfg['beta']}, "
                   f"sigma={cfg['sigma']}", "schedule": args.schedule, "sv_side": args.sv,
                   "parallelism": f"agents {N} over {world} GPU(s)" + (f", consensus: {args.comm}" if world > 1 else ""),
                   "l2": f"inputs > L2: K2 streams {lay['layout_bytes'] / 1e9:.2f} GB of records per iteration "
                         f"per GPU against a {l2_mb()} MB L2 (no flush needed)",
                   "final_relnorm": float(lg[-1, 0]) if len(lg) else None},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "mace_solve() on host float64 y/weights; includes H2D, solve, D2H image+stack"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / pk.get("hbm_gbs"), "traffic": k2_traffic(args.config, args.sv),
                     "kernel": "k_icd_sv (K2)", "records": "weighted" if plan.info().get("weighted") else "plain",
                     "bytes_per_launch": alg, "layout_bytes_per_launch": lay["layout_bytes"],
                     "k2_avg_ms": k2_avg_ms, "k2_share": k2_avg_ms * iters * args.steps / ms, "c_mean": lay["c_mean"],
                     "peak_source": "MEASURED_PEAKS.json" if not pk.get("_fallback") else "fallback"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "setup_s": {"scan": t_scan, "plan": t_plan},
    }
    if pnp:  # K5 alone: 17-layer CNN on the consensus image, CUDA events on the library stream
        reps = 20
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            den.device_apply(plan)
        e1.record(stream)
        barrier()
        k5_ms = e0.elapsed_time(e1) / reps
        flop = 2.0 * geom.n_pixels * 9 * (64 + 15 * 64 * 64 + 64)
        line["k5"] = {"kernel": "k_conv64_roll (tcgen05, layers 2-16) + k_conv_first + k_conv_last_roll", "ms_per_denoise": k5_ms,
                      "flop_per_denoise": flop, "achieved_tflops": flop / (k5_ms / 1e3) / 1e12,
                      "peak_tflops": pk.get("bf16_tflops"), "peak_source": "MEASURED_PEAKS bf16_tflops (burst: "
                      "timed alone)", "frac": flop / (k5_ms / 1e3) / 1e12 / pk.get("bf16_tflops", 1.0),
                      "frac_of_sustained": flop / (k5_ms / 1e3) / 1e12 / pk.get("bf16_tflops_sustained", 1.0),
                      "share_of_step": k5_ms * iters / (ms / args.steps)}
        line["config"]["workload"] = line["config"]["workload"].replace("qGGMRF beta", "PnP CNN denoiser (K5); beta")
        line["config"]["prior"] = "PnP: 17-layer 64-ch 3x3 CNN, He-normal(seed 0) x 0.1 weights in bf16, x - net(x)"
    if world == 1 and args.ttr_iters > 0 and not pnp:
        line["time_to_rmse_1e-3"] = time_to_rmse(plan, args.config, N, n, args.ttr_iters)
    elif world > 1 and args.ttr_iters > 0 and not pnp:
        path = os.path.join(ROOT, "tests", "golden", f"central_c{args.config}.npz")
        if os.path.exists(path):
            line["time_to_rmse_1e-3"] = time_to_rmse_ranks(mb, prob, mcfg, comm, np.load(path)["image"],
                                                           args.ttr_iters, ms / (args.steps * iters),
                                                           os.path.basename(path))
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.config, mats, y, lam, sample_iters=args.cpu_iters)
        ttr = line.get("time_to_rmse_1e-3") or {}
        if ttr.get("iterations"):
            per_iter = N * n / line["cpu_baseline"]["value"]
            line["cpu_baseline"]["time_to_rmse_1e-3_s_est"] = ttr["iterations"] * per_iter
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def time_to_rmse(plan, config, N, n, max_iters):
    """Device time until ||xbar_k - x*|| / ||x*|| <= 1e-3 and stays there, x* = the converged
    CPU-oracle MAP image (tests/golden/central_c{config}.npz).  Fresh solve from w = 0."""
    path = os.path.join(ROOT, "tests", "golden", f"central_c{config}.npz")
    if not os.path.exists(path):
        return None
    ref = np.load(path)["image"].astype(np.float32)
    plan.set_ref(ref)
    plan.stack_init(None, N)
    plan.states_from(0)
    ms = plan.iterate(max_iters, 0, 0.8, False, 1e-300, N, True)
    lg, _ = plan.read_log(max_iters)
    plan.set_ref(None)
    nr = lg[:, 3]
    ok = nr <= 1e-3
    first = None
    for i in range(len(nr)):
        if ok[i:].all():
            first = i + 1
            break
    return {"iterations": first, "seconds": None if first is None else ms / 1e3 * first / max_iters,
            "final_nrmse": float(nr[-1]), "ran_iterations": max_iters, "reference": os.path.basename(path),
            "note": "device time of a fresh solve; first iteration after which NRMSE stays <= 1e-3"}


def time_to_rmse_ranks(mb, prob, mcfg, comm, ref, max_iters, ms_per_iter, ref_name, backend=None):
    """N ranks: the iterations until the NRMSE against the reference image (the CPU-oracle MAP)
    stays <= 1e-3, from a fresh multi-rank solve through mace_solve with ref_image (the NRMSE of the
    global consensus image is computed on the host after every iteration, so that solve runs without
    the CUDA-graph blocks), times the device milliseconds per iteration of this run's timed region
    (max over ranks)."""
    import dataclasses

    ref = np.asarray(ref, np.float64)
    res = _solve_api_ref(mb, prob, dataclasses.replace(mcfg, max_outer=max_iters), comm, ref, backend)
    nr = np.array([r["nrmse"] for r in res.log.rows], dtype=np.float64)
    ok = nr <= 1e-3
    first = next((i + 1 for i in range(len(nr)) if ok[i:].all()), None)
    return {"iterations": first, "seconds": None if first is None else first * ms_per_iter / 1e3,
            "final_nrmse": float(nr[-1]) if len(nr) else None, "ran_iterations": len(nr),
            "reference": ref_name,
            "note": "iterations of a fresh multi-rank solve (NRMSE of the consensus image each iteration) x "
                    "device ms per iteration of the timed region; first iteration after which NRMSE stays <= 1e-3"}


def _solve_api_ref(mb, prob, cfg, comm, ref, backend=None):
    try:
        return mb.mace_solve(prob, cfg, comm=comm, ref_image=ref, _backend=backend)
    except mb.ConvergenceError as err:
        return err.last_iterate


def plan_stream(plan):
    import ctypes

    s = ctypes.c_void_p()
    plan.call("mace_ctx_stream", ctypes.byref(s))
    return s.value


def _solve_api(mb, prob, cfg, comm, denoiser=None, backend=None):
    try:
        if denoiser is not None:
            return mb.mace_pnp_solve(prob, cfg, comm=comm, denoiser=denoiser, _backend=backend)
        return mb.mace_solve(prob, cfg, comm=comm, _backend=backend)
    except mb.ConvergenceError as err:
        return err.last_iterate


def cpu_baseline(config, mats, y, lam, sample_iters=2, threads=None):
    """CPU oracle (restated reference hot loop, float64) on a bounded sample: `sample_iters`
    MACE iterations of the same workload, agents mapped over min(N, cores) threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    from paper_1911_09278_b200 import gen

    cfg = gen.CONFIGS[config]
    N = cfg["n_agents"]
    cores = os.cpu_count() or 1
    threads = threads or min(N, cores)
    ns = int(np.sqrt(mats[0].n_pixels))
    prior = O.Prior("qggmrf", cfg["beta"], 2.0, 1.2, 1.0, 0.01)
    agents = O.build_agents(mats, y, lam, N, cfg["sigma"], prior, ns, workers=threads)
    run = O.mace_run(agents, 1, 0.8, workers=threads)  # warm-up: initialisation + first iteration
    t0 = time.perf_counter()
    run = O.mace_run(agents, sample_iters, 0.8, w0=run.stack, workers=threads, resume=True)
    dt = time.perf_counter() - t0
    n = ns * ns
    return {"value": N * n * len(run.relnorms) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample_iters} MACE iterations of config {config} (N={N} agents, {n} px), "
                      f"oracle/sweep.c float64 raster ICD, {threads} threads; host has {cores} cores",
            "seconds": dt}


def reference_scan(config: int, workers: int | None = None):
    """The config's scan for the reference arm without this repo's CUDA library: the oracle's
    tracer (oracle.iter_system_matrix, bit-identical to the reference's build_system_matrix; SHA-256
    tests in tests/test_oracle_golden.py) and gen.make_scan's data recipe (same phantom, same
    scipy per-view product, same Poisson draw), so y and weights equal the GPU arm's."""
    import scipy.sparse as sp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    gen = load_gen()
    c = gen.CONFIGS[config]
    ns, nv, nc = c["n_side"], c["n_views"], c["n_channels"]
    pitch = 1.0 if config == 0 else gen.pitch_for(ns)
    mats = O.build_system_matrix_parallel(ns, pitch, nv, nc, pitch, workers)
    phantom = gen.ellipse_phantom(ns, pitch, c["n_ellipses"], seed=0)
    proj = np.stack([sp.csr_matrix((m.lens, m.cols, m.row_ptr), shape=(m.n_channels, m.n_pixels)) @ phantom
                     for m in mats])
    y, lam = gen.poisson_sinogram(proj, c["I0"], seed=1)
    return c, ns, mats, y, lam


def _libmace_loaded() -> bool:
    try:
        return "libmace_b200" in open("/proc/self/maps").read()
    except OSError:
        return False


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    cores = os.cpu_count() or 1
    t0 = time.time()
    cfg, ns, mats, y, lam = reference_scan(args.config, cores)
    N = cfg["n_agents"]
    threads = min(N, cores)
    prior = O.Prior("qggmrf", cfg["beta"], 2.0, 1.2, 1.0, 0.01)
    agents = O.build_agents(mats, y, lam, N, cfg["sigma"], prior, ns, workers=threads)
    del mats
    t_setup = time.time() - t0
    per_step = max(1, args.cpu_iters if args.config < 2 else 1)  # config 2: ~3 s per iteration on 16 cores
    run = O.mace_run(agents, 1, 0.8, workers=threads)  # the solve's initialisation and first iteration
    for _ in range(args.warmup):
        run = O.mace_run(agents, 1, 0.8, w0=run.stack, workers=threads, resume=True)
    t0 = time.perf_counter()
    done = 0
    for _ in range(args.steps):  # steady-state iterations of one continuing solve
        run = O.mace_run(agents, per_step, 0.8, w0=run.stack, workers=threads, resume=True)
        done += len(run.relnorms)
    dt = time.perf_counter() - t0
    n = ns * ns
    value = N * n * done / dt
    if _libmace_loaded():
        raise SystemExit("reference arm mapped libmace_b200.so")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded ellipse phantom, "
            "Poisson counts; gen.py recipe, oracle tracer)", "impl": "reference",
            "config": {"workload": f"BASELINE config {args.config}: {ns}^2, {y.shape[0]} views x {y.shape[1]} ch, "
                       f"N={N} agents; each step = {per_step} MACE iteration(s) of one continuing solve "
                       f"(bounded sample of the {cfg['iters']}-iteration solve)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{per_step} MACE iteration(s) per step, oracle/sweep.c float64 raster "
                                       f"ICD, agents over {threads} threads of {cores}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "libmace_b200_loaded": False, "setup_s": t_setup}
    print(json.dumps(line), flush=True)


def run_batch(args):
    """Config 4: 64 independent 512^2 slices sharing the operator, batched per agent."""
    import torch

    import paper_1911_09278_b200 as mb
    from paper_1911_09278_b200 import gen
    from paper_1911_09278_b200.engine import plan_for

    cfg = gen.CONFIGS[args.config]
    N, iters = cfg["n_agents"], args.iters or cfg["iters"]
    t0 = time.time()
    geom, mats, phantoms, ys, lams = gen.make_batch(args.config, n_slices=args.slices or None)
    S, n = len(ys), geom.n_pixels
    t_scan = time.time() - t0
    prior = mb.PriorParams("qggmrf", beta=cfg["beta"], p=2.0, q=1.2, T=1.0, sigma_x=0.01)
    subsets = mb.partition_views(geom.n_views, N)
    t0 = time.time()
    plan = plan_for(mats, [s.view_indices for s in subsets], schedule="sv", sv=args.sv, n_slices=S)
    t_plan = time.time() - t0
    plan.load_data(np.stack(ys), np.stack(lams))
    plan.set_prior(prior)
    plan.set_agent_params(-1, prior.beta / N, 1.0 / cfg["sigma"] ** 2, False)
    stream = torch.cuda.ExternalStream(plan_stream(plan), device="cuda:0")

    def solve():
        plan.stack_init(None, N)
        plan.states_from(0)
        plan.iterate(iters, 0, 0.8, False, 1e-300, N, False)

    for _ in range(args.warmup):
        solve()
    plan.k2_timing(True)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            solve()
        e1.record(stream)
        torch.cuda.synchronize()
    k2_ms, k2_n = plan.k2_timing(False)
    ms = e0.elapsed_time(e1)
    updates = N * n * S * iters * args.steps
    alg_single, lay = algorithmic_bytes_per_pass(plan, N)
    # B_upd = 8c/S + 16 + 12 R/n per slice-update
    alg = 8 * lay["nnz"] + S * (16 * n * N + 12 * lay["rows"])
    pk = peaks()
    k2_avg = k2_ms / max(k2_n, 1)
    achieved = alg / (k2_avg / 1e3) / 1e9
    probs = [mb.ReconProblem(geom, mats, ys[s], lams[s], prior) for s in range(S)]
    mcfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=cfg["sigma"], max_outer=iters, tol=1e-300, residuals="none",
                         sv_side=args.sv)
    def solve_batch():
        try:
            mb.mace_solve_batch(probs, mcfg)
        except mb.ConvergenceError:
            pass

    solve_batch()  # warm-up, as for the single-slice e2e (pinned result staging is allocated here)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(max(1, args.steps // 2)):
        solve_batch()
    e2e_s = (time.perf_counter() - t0) / max(1, args.steps // 2)
    line = {
        "metric": METRIC, "value": updates / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded per-slice ellipse phantoms; gen.make_batch)",
        "config": {"workload": f"BASELINE config {args.config}: {S} slices x {geom.n_side}^2, {geom.n_views} views x "
                   f"{geom.n_channels} ch, N={N} agents, {iters} iterations", "sv_side": args.sv,
                   "parallelism": f"{N} agents x {S} slices on 1 GPU"},
        "e2e": {"value": N * n * S * iters / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 2 * S * geom.n_views *
                geom.n_channels * 4, "d2h_bytes_per_step": S * (n + N * n) * 4,
                "note": "mace_solve_batch() on host arrays"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / pk.get("hbm_gbs"), "traffic": None, "kernel": "k_icd_sv (K2), slices batched",
                     "bytes_per_launch": alg, "k2_avg_ms": k2_avg, "k2_share": k2_ms / ms,
                     "note": "SURVEY 8(d) counts A once per launch for the 64 slices that share it (B_upd = 8c/64 + "
                             "16 + 12 R/n), so the HBM fraction is nominal; per slice the kernel streams the A "
                             "records from L2 and is bound by the L1 data pipe like config 1 (k2_ms_per_slice)",
                     "k2_ms_per_slice": k2_avg / S},
        "gpu_launches": (3 + 4 * iters) * args.steps, "clocks": clk.summary(),
        "setup_s": {"scan": t_scan, "plan": t_plan},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--schedule", default="sv", choices=["sv", "raster"])
    ap.add_argument("--sv", type=int, default=8)
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ttr-iters", type=int, default=-1,
                    help="iterations for time-to-RMSE (0: skip; default: per config, TTR_ITERS)")
    ap.add_argument("--slices", type=int, default=0, help="config 4: number of slices (default 64)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: consensus by an NCCL all-reduce on the library stream, or by the library's own "
                         "push/reduce kernels over NVLink peer memory (PeerComm)")
    ap.add_argument("--cpu-test", action="store_true", help=argparse.SUPPRESS)  # tests: gloo ranks on CPU
    args = ap.parse_args()
    if args.ttr_iters < 0:
        args.ttr_iters = 0 if args.cpu_test else TTR_ITERS.get(args.config, 0)
    if args.impl == "ours":
        cmd = launch_command(args.gpus, sys.argv[1:])
        if cmd is not None:  # one process per GPU: re-run this script under torchrun
            sys.stdout.flush()
            os.execv(cmd[0], cmd)
    if args.impl == "reference":
        run_reference(args)
    elif args.cpu_test:
        run_cpu_test(args)
    elif args.config == 4:
        run_batch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
