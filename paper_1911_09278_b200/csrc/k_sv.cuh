// K2, super-voxel schedule: the partial-update ICD pass of every local agent.
//
// Restates _sweep (pkg/src/macetomo/icd.py:67-139) per tile, with the
// consensus reflection v = 2 G(w) - w (mace.py:99-102) fused into the
// prologue and the Mann step w <- rho (2X - v) + (1 - rho) w (mace.py:111-117)
// fused into the epilogue.
//
// One warp owns one (agent, super-voxel) work item at a time, pulled from a
// global queue in colour-class order.  Per item:
//   1. the tile's error-sinogram band (one 16-byte-aligned window of {e, lambda}
//      rows per view) is staged in shared memory by TMA bulk copies
//      (cp.async.bulk ... mbarrier::complete_tx), one copy per view;
//   2. the tile's state (+ 1-pixel halo), theta2, w and G(w) come in with
//      unrolled independent loads, and the first D columns of A are already in
//      flight (128-bit streaming loads, evict-first);
//   3. the S*S pixels are updated sequentially (tile-raster order) against the
//      staged band: theta1 gather, fused qGGMRF 8-neighbour surrogate, a single
//      two-value warp reduction (numerator, denominator), 1-D solve, scatter;
//   4. the band's net change is folded back into global e with red.add, and the
//      tile's z / w (Mann) and norm partials are written.
//
// Column storage (layout.cpp): groups of 128 entries; inside a group of Lg
// entries slot 4l+q holds entry l + q*ceil(Lg/4), pads hold value 0 and the
// tile's dummy band row B (zeroed here), so the gather and the scatter run
// without predicates and lanes touch consecutive entries at each step.
#pragma once
#include "kernels.cuh"

namespace mace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// shared-memory bytes per warp for tile side S, band capacity `cap` rows, `vcap` views
__host__ __device__ constexpr size_t sv_warp_bytes(int S, int cap, int vcap)
{
    return 16 + 8 * (size_t)vcap + 12 * (size_t)cap + 4 * (size_t)((((S + 2) * (S + 2)) + 3) & ~3) +
           20 * (size_t)S * S;
}

__device__ __forceinline__ float fast_exp2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// qGGMRF neighbour term with the 8 lanes' shared subexpressions fused (icd.py:45-64):
// returns c = w rho'(d)/d (surrogate coefficient) and g = w rho'(d), MUFU log2/exp2.
template <bool kP2>
__device__ __forceinline__ void qg_term(float d, float wk, const PriorC& P, float& g, float& c)
{
    const float ad = fabsf(d);
    if (kP2) {
        // p = 2: rho'(d) = d * k(|d|), rho'(d)/d = k(|d|), k = sx^-2 um (q/2 + um) / (1 + um)^2
        float k;
        if (ad <= P.floor_) {
            k = P.inv_sx2;  // exact p = 2 limit below the floor (icd.py:58-60)
        } else {
            const float um = fast_exp2(P.qmp * __log2f(ad * P.inv_Tsx));
            const float opu = 1.0f + um;
            k = __fdividef(P.inv_sxp * um * (P.qp + um), opu * opu);
        }
        c = wk * k;
        g = c * d;
    } else {
        g = wk * qg_influence(d, P);
        c = wk * qg_coef(d, P);
    }
}

// Two half-warp sub-chains per tile: half 0 walks the top S/2 rows, half 1 the
// bottom S/2 rows (never 8-neighbours), one pixel each per step; 16 lanes x 8
// slots cover a 128-entry column group.  Within a step the two pixels see each
// other's previous-step updates only (the scatter is two-phase: half 0 writes,
// then half 1 re-reads and writes), so shared rows are never lost.
template <int S, int D, bool kP2>
__global__ void __launch_bounds__(128, 4) k_icd_sv(PassParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    if (P.done && *P.done) return;
    constexpr int SS = S * S, HS = SS / 2, S2 = S + 2, T2 = S2 * S2, T2p = (T2 + 3) & ~3;
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const int cap = P.band_cap, vcap = P.view_cap;
    unsigned char* base = smem + (threadIdx.x >> 5) * sv_warp_bytes(S, cap, vcap);
    uint64_t* bar = reinterpret_cast<uint64_t*>(base);
    int2* sbt = reinterpret_cast<int2*>(base + 16);
    float2* sel = reinterpret_cast<float2*>(base + 16 + 8 * (size_t)vcap);
    float* se0 = reinterpret_cast<float*>(sel + cap);
    float* zt = se0 + cap;
    float* svv = zt + T2p;
    float* sth = svv + SS;
    float* swo = sth + SS;
    int2* spe = reinterpret_cast<int2*>(swo + SS);
    const int n = P.n_side;
    const PriorC& PR = P.pr;
    const bool quad = PR.kind == 0;
    // lanes hl = 0..7 of each half own the 8 neighbours (models.py:50-52 order)
    const int kk = hl & 7;
    const int ndr = c_dr[kk], ndc = c_dc[kk];
    const float nwk = hl < 8 ? c_nw[kk] : 0.f;
    const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;

    if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;

    for (;;) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(P.head, 1u);
        item = __shfl_sync(FULL, item, 0);
        if (item >= (unsigned)P.n_items) break;
        const uint32_t code = __ldg(P.queue + item);
        const AgentDev& A = P.agents[code >> kAgentShift];
        const int sv = (int)(code & kSvMask);
        float2* __restrict__ el = A.el;
        float* __restrict__ z = A.z;
        float* __restrict__ w = A.w;
        const int V = A.V;
        const int nsv = A.n_sv_side;
        const int r0 = (sv / nsv) * S, c0 = (sv % nsv) * S;
        const float beta = A.beta_eff, inv_s2 = A.inv_s2;
        const int clamp = A.clamp;
        const int2* bt = A.band + (size_t)sv * V;
        const int B = __ldg(A.bsize + sv);
        const uint32_t dummy2 = (uint32_t)B | ((uint32_t)B << 16);

        // -- 1. band table, then the band: one TMA bulk copy per view (P.stage_tma), or
        //       16-byte LDGSTS (cp.async.cg, L2-coherent) with a quarter-warp per view
        for (int j = lane; j < V; j += 32) sbt[j] = __ldg(bt + j);
        if (P.stage_tma) {
            fence_proxy_async();  // order earlier generic accesses of the band before the async-proxy writes
            __syncwarp();
            if (lane == 0) mbar_expect_tx(bar, (uint32_t)B * 8u);
            for (int j = lane; j < V; j += 32) {
                const int2 b = sbt[j];
                const int cnt = b.y & 0xffff;
                if (cnt) bulk_g2s(sel + (b.y >> 16), el + b.x, (uint32_t)cnt * 8u, bar);
            }
        } else {
            __syncwarp();
            for (int j = lane >> 3; j < V; j += 4) {
                const int2 b = sbt[j];
                const int cnt = b.y & 0xffff, pos = b.y >> 16;
                for (int c2 = 2 * (lane & 7); c2 < cnt; c2 += 16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sel + pos + c2)),
                                 "l"(el + b.x + c2)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // -- 2. tile state + halo, column table, theta2, w and v = 2 G(w) - w
#pragma unroll
        for (int i0 = 0; i0 < T2p; i0 += 32) {
            const int i = i0 + lane;
            if (i < T2) {
                const int rr = r0 - 1 + i / S2, cc = c0 - 1 + i % S2;
                zt[i] = (rr >= 0 && rr < n && cc >= 0 && cc < n) ? __ldcg(z + (size_t)rr * n + cc) : 0.f;
            }
        }
#pragma unroll
        for (int i0 = 0; i0 < SS; i0 += 32) {
            const int i = i0 + lane;
            if (i < SS) {
                const int rr = r0 + i / S, cc = c0 + i % S;
                spe[i] = __ldg(A.pix + (size_t)sv * SS + i);
                if (rr < n && cc < n) {
                    const size_t s = (size_t)rr * n + cc;
                    sth[i] = A.th[s];
                    const float wo = w[s];
                    swo[i] = wo;
                    svv[i] = P.mode ? 2.f * __ldg(P.g + (size_t)A.slice * n * n + s) - wo : A.vt[s];
                } else {
                    sth[i] = 0.f;
                    svv[i] = 0.f;
                    swo[i] = 0.f;
                }
            }
        }
        __syncwarp();

        // -- 3. sequential pixel loop (two sub-chains); the first 128 entries of each
        //       column are streamed D steps ahead, longer columns (rare) take a tail
        const float* __restrict__ av = A.val;
        const uint16_t* __restrict__ ai = A.idx;
        float4 va[D], vb[D];
        uint4 ix[D];
        auto fetch = [&](int k, float4& a4, float4& b4, uint4& i8) {
            a4 = make_float4(0.f, 0.f, 0.f, 0.f);
            b4 = a4;
            i8 = make_uint4(dummy2, dummy2, dummy2, dummy2);
            if (k < HS) {
                const int2 pe = spe[k + half * HS];
                if (8 * hl < min(pe.y, 128)) {
                    a4 = __ldcs(reinterpret_cast<const float4*>(av + pe.x + 8 * hl));
                    b4 = __ldcs(reinterpret_cast<const float4*>(av + pe.x + 8 * hl + 4));
                    i8 = __ldcs(reinterpret_cast<const uint4*>(ai + pe.x + 8 * hl));
                }
            }
        };
#pragma unroll
        for (int u = 0; u < D; ++u) fetch(u, va[u], vb[u], ix[u]);
        if (P.stage_tma) {
            while (!mbar_try_wait(bar, phase)) {
            }
            phase ^= 1u;
        } else {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
        }
        for (int f = lane; f < B; f += 32) se0[f] = sel[f].x;
        if (lane == 0) sel[B] = make_float2(0.f, 0.f);  // the pads' dummy row
        __syncwarp();

        double dsq = 0.0;
#pragma unroll 1
        for (int kb = 0; kb < HS; kb += D) {
#pragma unroll
            for (int u = 0; u < D; ++u) {
                const int k = kb + u;
                if (k < HS) {
                    const int p = k + half * HS;
                    const int lr = p / S, lc = p % S;
                    const bool inside = (r0 + lr < n) && (c0 + lc < n);
                    const int2 pe = spe[p];
                    const int ci = (lr + 1) * S2 + (lc + 1);
                    const float zs = zt[ci];
                    const float vv[8] = {va[u].x, va[u].y, va[u].z, va[u].w, vb[u].x, vb[u].y, vb[u].z, vb[u].w};
                    const uint32_t ii[8] = {ix[u].x & 0xffffu, ix[u].x >> 16, ix[u].y & 0xffffu, ix[u].y >> 16,
                                            ix[u].z & 0xffffu, ix[u].z >> 16, ix[u].w & 0xffffu, ix[u].w >> 16};
                    float2 xs[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) xs[q] = sel[ii[q]];
                    float num = 0.f;
#pragma unroll
                    for (int q = 0; q < 8; ++q) num = fmaf(vv[q] * xs[q].y, xs[q].x, num);
                    if (pe.y > 128) {  // rare long column: remaining groups
                        for (int g0 = 128; g0 < pe.y; g0 += 128) {
                            if (8 * hl < min(pe.y - g0, 128)) {
                                const float4 a4 = *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl);
                                const float4 b4 = *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl + 4);
                                const uint4 q8 = *reinterpret_cast<const uint4*>(ai + pe.x + g0 + 8 * hl);
                                const float v2[8] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
                                const uint32_t i2[8] = {q8.x & 0xffffu, q8.x >> 16, q8.y & 0xffffu, q8.y >> 16,
                                                        q8.z & 0xffffu, q8.z >> 16, q8.w & 0xffffu, q8.w >> 16};
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    const float2 x = sel[i2[q]];
                                    num = fmaf(v2[q] * x.y, x.x, num);
                                }
                            }
                        }
                    }
                    // prior: lanes hl < 8, neighbour kk of this half's pixel (weight 0 elsewhere)
                    float den;
                    {
                        const int gr = r0 + lr + ndr, gc = c0 + lc + ndc;
                        const bool valid = gr >= 0 && gr < n && gc >= 0 && gc < n && beta > 0.f;
                        const float wk = valid ? nwk : 0.f;
                        const float zr = zt[(lr + 1 + ndr) * S2 + (lc + 1 + ndc)];
                        float g, c;
                        if (quad) {
                            g = wk * (zs - zr);
                            c = wk;
                        } else {
                            qg_term<kP2>(zs - zr, wk, PR, g, c);
                        }
                        num -= beta * g;
                        den = beta * c;
                    }
#pragma unroll
                    for (int o = 8; o; o >>= 1) {
                        num += __shfl_xor_sync(FULL, num, o);
                        den += __shfl_xor_sync(FULL, den, o);
                    }
                    // 1-D solve (icd.py:128-134); the reference skips pixels with den <= 0
                    if (quad && beta > 0.f) {
                        num -= beta * PR.eps2 * zs;
                        den += beta * PR.eps2;
                    }
                    num -= inv_s2 * (zs - svv[p]);
                    den += sth[p] + inv_s2;
                    float alpha = (inside && den > 0.f) ? __fdividef(num, den) : 0.f;
                    if (clamp && zs + alpha < 0.f) alpha = -zs;
                    zt[ci] = zs + alpha;
                    dsq += (double)alpha * alpha;
                    // two-phase scatter: half 0 writes, half 1 re-reads and writes
                    if (half == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) sel[ii[q]].x = xs[q].x - alpha * vv[q];
                    }
                    if (pe.y > 128 && half == 0) {
                        for (int g0 = 128; g0 < pe.y; g0 += 128) {
                            if (8 * hl < min(pe.y - g0, 128)) {
                                const float4 a4 = *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl);
                                const float4 b4 = *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl + 4);
                                const uint4 q8 = *reinterpret_cast<const uint4*>(ai + pe.x + g0 + 8 * hl);
                                const float v2[8] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
                                const uint32_t i2[8] = {q8.x & 0xffffu, q8.x >> 16, q8.y & 0xffffu, q8.y >> 16,
                                                        q8.z & 0xffffu, q8.z >> 16, q8.w & 0xffffu, q8.w >> 16};
#pragma unroll
                                for (int q = 0; q < 8; ++q) sel[i2[q]].x -= alpha * v2[q];
                            }
                        }
                    }
                    __syncwarp();
                    if (half == 1) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) sel[ii[q]].x -= alpha * vv[q];
                        if (pe.y > 128) {
                            for (int g0 = 128; g0 < pe.y; g0 += 128) {
                                if (8 * hl < min(pe.y - g0, 128)) {
                                    const float4 a4 = *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl);
                                    const float4 b4 =
                                        *reinterpret_cast<const float4*>(av + pe.x + g0 + 8 * hl + 4);
                                    const uint4 q8 = *reinterpret_cast<const uint4*>(ai + pe.x + g0 + 8 * hl);
                                    const float v2[8] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
                                    const uint32_t i2[8] = {q8.x & 0xffffu, q8.x >> 16, q8.y & 0xffffu,
                                                            q8.y >> 16, q8.z & 0xffffu, q8.z >> 16,
                                                            q8.w & 0xffffu, q8.w >> 16};
#pragma unroll
                                    for (int q = 0; q < 8; ++q) sel[i2[q]].x -= alpha * v2[q];
                                }
                            }
                        }
                    }
                    __syncwarp();
                }
                fetch(k + D, va[u], vb[u], ix[u]);
            }
        }
        dsq += __shfl_xor_sync(FULL, dsq, 16);  // the two sub-chains
        __syncwarp();

        // -- 4. fold the band's net change into global e (one 16-byte vector red per row
        //       pair: {de0, 0, de1, 0} onto {e0, lambda0, e1, lambda1}); z, Mann, norms
        for (int j = lane >> 3; j < V; j += 4) {
            const int2 b = sbt[j];
            const int cnt = b.y & 0xffff, pos = b.y >> 16;
            for (int c2 = 2 * (lane & 7); c2 < cnt; c2 += 16) {
                const float d0 = sel[pos + c2].x - se0[pos + c2];
                const float d1 = sel[pos + c2 + 1].x - se0[pos + c2 + 1];
                if (d0 != 0.f || d1 != 0.f)
                    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(el + b.x + c2),
                                 "f"(d0), "f"(0.f), "f"(d1), "f"(0.f)
                                 : "memory");
            }
        }
        double dw2 = 0.0, wn2 = 0.0, wo2 = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < SS; i0 += 32) {
            const int i = i0 + lane;
            const int rr = r0 + i / S, cc = c0 + i % S;
            if (i < SS && rr < n && cc < n) {
                const size_t s = (size_t)rr * n + cc;
                const float zn = zt[(i / S + 1) * S2 + (i % S + 1)];
                __stcg(z + s, zn);
                if (P.mode) {
                    const float wo = swo[i];
                    const float wn = P.rho * (2.f * zn - svv[i]) + (1.f - P.rho) * wo;
                    w[s] = wn;
                    const double dd = (double)wn - (double)wo;
                    dw2 += dd * dd;
                    wn2 += (double)wn * wn;
                    wo2 += (double)wo * wo;
                }
            }
        }
        dw2 = warp_sum_d(dw2);
        wn2 = warp_sum_d(wn2);
        wo2 = warp_sum_d(wo2);
        if (lane == 0) {
            double* o = P.part + (size_t)item * 4;
            o[0] = dsq;
            o[1] = dw2;
            o[2] = wn2;
            o[3] = wo2;
        }
        __syncwarp();
    }
    (void)hmask;
}

}  // namespace mace
