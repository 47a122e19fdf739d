"""K5 (tcgen05 implicit-GEMM CNN denoiser) against the torch CPU oracle (oracle/cnn.py),
and MACE-PnP with it (BASELINE config 3 recipe) against the oracle loop with the same
callable.

Tolerances: the GPU accumulates in fp32 and both sides round activations to bf16 between
layers, so an activation can land one bf16 ulp (2^-8 relative) apart when the fp32 sum
straddles a rounding boundary.  The residual net(x) is checked to 2e-2 relative (L2) and the
denoised image x - net(x) to 1e-4 relative."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from cnn import cnn_apply

import paper_1911_09278_b200 as mb
from paper_1911_09278_b200 import gen
from paper_1911_09278_b200.denoisers import CnnDenoiser, cnn_weights

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def _net(x, out):
    """net(x) = x32 - H(x): the GPU applies the residual to the fp32 input."""
    return np.asarray(x, np.float32).astype(np.float64) - out


@pytest.mark.parametrize("n_side,seed", [(64, 0), (512, 1), (200, 2), (130, 3)])
def test_cnn_matches_cpu_oracle(n_side, seed):
    """He-normal weights at unit scale so every layer's activations are O(1) and the
    residual net(x) is O(x): a wrong descriptor, tap or channel mapping cannot hide."""
    rng = np.random.default_rng(seed)
    x = rng.random(n_side * n_side)
    w = cnn_weights(seed, scale=1.0)
    H = CnnDenoiser(n_side, weights=w)
    out = H(x)
    ref = cnn_apply(np.asarray(x, np.float32), w, n_side)
    r_gpu, r_ref = _net(x, out), np.asarray(x, np.float32) - ref
    assert rel(r_ref, x) > 0.05
    print(f"n={n_side}: K5 {H.last_ms:.3f} ms, net rel err {rel(r_gpu, r_ref):.2e}, "
          f"max abs {np.max(np.abs(r_gpu - r_ref)):.2e} of max {np.max(np.abs(r_ref)):.2e}")
    # bf16 activations: fp32 sums that straddle a rounding boundary land one bf16 ulp apart,
    # and such differences compound over 17 random layers -> a few percent, not a bug signal
    # (the exact-arithmetic test below pins the tap / channel / padding mapping bit for bit)
    assert rel(r_gpu, r_ref) < 4e-2, rel(r_gpu, r_ref)


# 16 and 40: one output row per CTA; 200 and 300: short row runs; 512: 14 rows (the rolling accumulators
# wrap once); 1024: 57 rows per CTA (seven wraps)
@pytest.mark.parametrize("n_side,seed", [(16, 14), (40, 15), (64, 11), (200, 12), (300, 17), (512, 13), (1024, 16)])
def test_cnn_exact_taps_channels_padding(n_side, seed):
    """Every middle layer is a single 3x3 tap and a channel permutation (one nonzero product per
    output), so both sides compute exactly: the GPU must reproduce the oracle bit for bit,
    which pins the UMMA descriptors (tap shift, channel groups), the TMA zero padding and the
    TMEM -> NHWC epilogue."""
    rng = np.random.default_rng(seed)
    C = 64
    w = [np.zeros((C, 1, 3, 3), np.float32)]
    w[0][:, 0, 1, 1] = rng.choice([0.5, 1.0, 2.0], C)  # layer 1: scaled copies of x
    for _ in range(15):
        m = np.zeros((C, C, 3, 3), np.float32)
        t = rng.integers(9)
        perm = rng.permutation(C)
        m[np.arange(C), perm, t // 3, t % 3] = rng.choice([0.5, 1.0, 2.0], C)
        w.append(m)
    last = np.zeros((1, C, 3, 3), np.float32)
    last[0, rng.integers(C), 1, 1] = 1.0
    w.append(last)
    x = rng.integers(0, 256, n_side * n_side).astype(np.float64) / 256.0
    out = CnnDenoiser(n_side, weights=w)(x)
    ref = cnn_apply(np.asarray(x, np.float32), w, n_side)
    assert np.array_equal(np.asarray(out, np.float32), np.asarray(ref, np.float32))


def _bf16_rne_f64(v):
    """exact fp64 -> bf16 round-to-nearest-even (no double rounding through fp32)"""
    m, e = np.frexp(v)
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)


@pytest.mark.parametrize("h,w,layer,seed", [(128, 128, 0, 21), (96, 200, 14, 22), (33, 130, 7, 23)])
def test_cnn_one_layer_bf16_rounding(h, w, layer, seed):
    """One 64->64 layer alone (tcgen05 UMMAs, fp32 accumulation in TMEM, ReLU, bf16 epilogue) on a
    fixed bf16 input against the exact fp64 conv rounded once to bf16.  At least 99.9% of the
    outputs must be bit-identical and every other one explained by one fp32 accumulation plus one
    rounding: one bf16 ulp away and
    a near-tie: the exact value within the fp32 accumulation bound (576 terms x 2^-24 x sum|terms|)
    of the midpoint between its two bf16 neighbours, or (more than one ulp) an output that cancels
    far below its terms, where the fp32 bound exceeds the output's own ulp.  A wrong tap, channel,
    K-step or fragment order would break the count by orders of magnitude."""
    from paper_1911_09278_b200.denoisers import from_bf16_bits, to_bf16_bits

    rng = np.random.default_rng(seed)
    wts = cnn_weights(seed, scale=1.0)
    Wl = wts[1 + layer].astype(np.float64)  # (64 oc, 64 ic, 3, 3), bf16 values
    x_bits = to_bf16_bits(rng.random((64, h, w)).astype(np.float32))
    x = from_bf16_bits(x_bits).astype(np.float64)
    xp = np.zeros((64, h + 2, w + 2))
    xp[:, 1:-1, 1:-1] = x
    exact = np.zeros((64, h, w))
    mag = np.zeros((64, h, w))
    for dy in range(3):
        for dx in range(3):
            sh = xp[:, dy:dy + h, dx:dx + w].reshape(64, -1)
            exact += (Wl[:, :, dy, dx] @ sh).reshape(64, h, w)
            mag += (np.abs(Wl[:, :, dy, dx]) @ np.abs(sh)).reshape(64, h, w)
    ref = _bf16_rne_f64(np.maximum(exact, 0.0))
    got = from_bf16_bits(CnnDenoiser(h, weights=wts).layer(layer, x_bits)).astype(np.float64)
    same = got == ref
    frac = same.mean()
    bad = ~same
    ulp = np.ldexp(1.0, np.frexp(np.maximum(np.abs(ref), 1e-30))[1] - 8)
    bound = 576 * 2.0 ** -24 * mag
    relu = bad & ((got == 0) | (ref == 0))  # fp32 sum and exact value on either side of the ReLU
    rnd = bad & ~relu
    ulps = np.abs(got - ref)[rnd] / ulp[rnd]
    mid = np.minimum(got, ref)[rnd] + 0.5 * np.abs(got - ref)[rnd]
    tie = np.abs(exact[rnd] - mid) / bound[rnd]
    print(f"layer {layer} {h}x{w}: {frac * 100:.4f}% bit-identical; {rnd.sum()} rounding and {relu.sum()} ReLU "
          f"mismatches; max {ulps.max() if ulps.size else 0:.3f} ulp; midpoint distance / fp32 bound max "
          f"{tie.max() if tie.size else 0:.3e}; ReLU mismatch / bound max "
          f"{(np.abs(got - ref)[relu] / bound[relu]).max() if relu.any() else 0:.3e}")
    assert frac >= 0.999, frac
    # every mismatch is one fp32 accumulation (|sum - exact| <= bound) plus one rounding to bf16
    ulp_got = np.ldexp(1.0, np.frexp(np.maximum(np.abs(got), 1e-30))[1] - 8)
    assert np.all((np.abs(got - exact.clip(min=0.0)) <= 0.5 * ulp_got + bound)[bad])
    # more than one ulp apart only where the output cancels far below its terms (bound >= ulp)
    far = np.zeros_like(bad)
    far[rnd] = ulps > 1.0 + 1e-6
    assert np.all(bound[far] >= ulp[far]), (bound[far] / ulp[far]).min()
    # the one-ulp ones sit next to the midpoint between their two bf16 neighbours
    assert np.all(tie[ulps <= 1.0 + 1e-6] <= 1.0)


def test_cnn_config3_weights_run():
    """The literal BASELINE config-3 weights (He-normal x 0.1 per layer) shrink the residual
    by ~0.1 per layer, so H is the identity to fp32 precision: check exactly that."""
    n = 512
    x = np.random.default_rng(9).random(n * n) * 0.03
    out = CnnDenoiser(n, weights=cnn_weights(0))(x)
    assert np.allclose(out, np.asarray(x, np.float32), rtol=1e-6, atol=0)


def test_mace_pnp_with_cnn_denoiser_vs_oracle_loop():
    """Config-3 recipe in miniature: PnP agents at sqrt(N) sigma, beta = 0, H = the CNN."""
    ns, nv, nc, N = 64, 90, 91, 4
    pitch = 128.0 / ns
    geom = mb.Geometry(ns, pitch, nv, nc, pitch)
    mats = mb.build_system_matrix(geom)
    ph = gen.ellipse_phantom(ns, pitch, 10, seed=0)
    y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 1e4, seed=1)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", 25.0, 2.0, 1.2, 1.0, 0.01))
    w = cnn_weights(3, scale=0.5)
    H = CnnDenoiser(ns, weights=w)
    sigma, iters = 2e-4, 20
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=sigma, mode="pnp", denoiser=mb.DenoiserSpec("identity"),
                        max_outer=iters, tol=1e-300, residuals="none", schedule="raster")
    try:
        res = mb.mace_pnp_solve(prob, cfg, denoiser=H)
    except mb.ConvergenceError as err:
        res = err.last_iterate
    agents = O.build_agents(mats, y, lam, N, sigma, O.Prior("qggmrf", 25.0, 2.0, 1.2, 1.0, 0.01), ns, pnp=True)
    run = O.mace_run(agents, iters, 0.8, denoiser=lambda v: cnn_apply(v, w, ns))
    assert rel(res.image, run.image) < 1e-4


def test_pnp_denoiser_in_device_loop_matches_host_steps():
    """mace_iterate(use_g=2) applies the CNN inside the device loop; the same CNN driven as a plain
    host callable (one iteration per call, H on the host boundary) must give the same iterates."""
    ns, nv, nc, N = 64, 90, 91, 4
    pitch = 128.0 / ns
    geom = mb.Geometry(ns, pitch, nv, nc, pitch)
    mats = mb.build_system_matrix(geom)
    ph = gen.ellipse_phantom(ns, pitch, 10, seed=2)
    y, lam = gen.poisson_sinogram(gen.host_forward_project(mats, ph), 1e4, seed=3)
    prob = mb.ReconProblem(geom, mats, y, lam, mb.PriorParams("qggmrf", 25.0, 2.0, 1.2, 1.0, 0.01))
    w = cnn_weights(5, scale=0.5)
    H = CnnDenoiser(ns, weights=w)
    cfg = mb.MaceConfig(n_subsets=N, rho=0.8, sigma=2e-4, mode="pnp", denoiser=mb.DenoiserSpec("identity"),
                        max_outer=15, tol=1e-300, residuals="none", schedule="raster")

    def solve(den):
        try:
            return mb.mace_pnp_solve(prob, cfg, denoiser=den)
        except mb.ConvergenceError as err:
            return err.last_iterate

    dev = solve(H)
    host = solve(lambda v: H(v))  # no device hooks: host round trip every iteration
    assert rel(dev.image, host.image) < 1e-6
    assert rel(dev.stack, host.stack) < 1e-6


@pytest.mark.parametrize("n_side", [200, 512])
def test_cnn_is_bitwise_repeatable(n_side):
    """The rolling-accumulator layers reuse 8 TMEM slots and 8 halo slots behind mbarriers; a missing wait would
    show up as run-to-run differences on random unit-scale weights.  30 denoises must be bit-identical."""
    rng = np.random.default_rng(41)
    x = rng.random(n_side * n_side)
    den = CnnDenoiser(n_side, weights=cnn_weights(41, scale=1.0))
    first = den(x)
    for _ in range(29):
        assert np.array_equal(den(x), first)


@pytest.mark.parametrize("n_side", [64, 200, 512])
def test_cnn_launch_variants_are_bit_identical(n_side, monkeypatch):
    """The middle layers as 15 launches or as one persistent launch (MACE_K5_SEQ), and the last layer
    on the tensor cores or on the CUDA cores (MACE_K5_LAST): the persistent kernel runs the same
    UMMAs, so it must match the per-layer launches bit for bit; the two last-layer kernels sum the
    576 products in different orders (fp32), so they agree to fp32 rounding."""
    rng = np.random.default_rng(31)
    x = rng.random(n_side * n_side)
    w = cnn_weights(31, scale=1.0)
    outs = {}
    monkeypatch.setenv("MACE_K5_ROWS", "2")  # the persistent kernel runs row pairs
    for seq in ("0", "1"):
        for last in ("tc", "fma"):
            monkeypatch.setenv("MACE_K5_SEQ", seq)
            monkeypatch.setenv("MACE_K5_LAST", last)
            outs[(seq, last)] = CnnDenoiser(n_side, weights=w)(x)
    assert np.array_equal(outs[("1", "tc")], outs[("0", "tc")])
    assert np.array_equal(outs[("1", "fma")], outs[("0", "fma")])
    r_tc, r_fma = _net(x, outs[("0", "tc")]), _net(x, outs[("0", "fma")])
    assert rel(r_tc, r_fma) < 1e-5
    monkeypatch.setenv("MACE_K5_LAST", "roll")  # layer 17 with rolling accumulators (k_conv_last_roll, the default)
    assert rel(_net(x, CnnDenoiser(n_side, weights=w)(x)), r_tc) < 1e-5
    # row units per MMA batch (MACE_K5_ROWS; 0 = one halo row at a time into rolling accumulators):
    # each output row receives the same UMMAs in another
    # order (fp32 accumulation), and one-ulp bf16 differences compound over 17 random unit-scale
    # layers -- so single rows, pairs and triples are each held to the CPU oracle like the default
    # (test_cnn_matches_cpu_oracle), and to each other at that level
    monkeypatch.setenv("MACE_K5_SEQ", "0")
    monkeypatch.setenv("MACE_K5_LAST", "tc")
    ref = np.asarray(x, np.float32) - cnn_apply(np.asarray(x, np.float32), w, n_side)
    units = {}
    for r in ("0", "1", "2", "3"):  # "0": rolling accumulators (k_conv64_roll, the default)
        monkeypatch.setenv("MACE_K5_ROWS", r)
        units[r] = _net(x, CnnDenoiser(n_side, weights=w)(x))
        assert rel(units[r], ref) < 4e-2, (r, rel(units[r], ref))
    assert rel(units["2"], units["3"]) < 4e-2 and rel(units["1"], units["3"]) < 4e-2
    assert rel(units["0"], units["3"]) < 4e-2
    # the rolling-accumulator layers as one cooperative launch with a grid-wide counter between layers
    # (MACE_K5_SEQ=1 with MACE_K5_ROWS=0): the same UMMAs in the same order, so bit-identical, twice in a
    # row (the counter runs on from denoise to denoise)
    monkeypatch.setenv("MACE_K5_ROWS", "0")
    monkeypatch.setenv("MACE_K5_SEQ", "0")
    one = CnnDenoiser(n_side, weights=w)(x)
    monkeypatch.setenv("MACE_K5_SEQ", "1")
    den = CnnDenoiser(n_side, weights=w)
    assert np.array_equal(den(x), one) and np.array_equal(den(x), one)
    # ... and pipelined (MACE_K5_SEQ=2, k_conv64_pipe): row runs shifted by half a run in odd layers, per-row
    # flags instead of any grid-wide wait; every output row still receives the same UMMAs in the same order
    monkeypatch.setenv("MACE_K5_SEQ", "2")
    den = CnnDenoiser(n_side, weights=w)
    assert np.array_equal(den(x), one) and np.array_equal(den(x), one) and np.array_equal(den(x), one)
