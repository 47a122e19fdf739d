// K2, super-voxel schedule: the partial-update ICD pass of every local agent.
//
// Restates _sweep (pkg/src/macetomo/icd.py:67-139) per tile, with the consensus
// reflection v = 2 G(w) - w (mace.py:99-102) fused into the prologue and the Mann step
// w <- rho (2X - v) + (1 - rho) w (mace.py:111-117) fused into the epilogue.
//
// One warp owns one (agent, super-voxel) work item at a time, pulled from a global queue in
// colour-class order, and updates every pixel of the tile once (Gauss-Seidel inside the tile).
// Lane-per-view mapping (layout.cpp): view j of the agent belongs to lane j % 32, group j / 32.
//
//  * The band windows of the lane's views (the error-sinogram rows the tile touches) live in the
//    lane's own shared-memory bank (planes e, lambda and a copy e0 of e): every gather and
//    scatter is bank-conflict free and lane-private.
//  * Pixels are visited in batches of four pixels of one parity class (internal.h): they are
//    never 8-neighbours, so the four prior terms are computed at once on lanes 8p..8p+7, and the
//    data terms theta1_p = sum a_p lambda e are gathered against the band as it stood before the
//    batch.  The exact sequential (Gauss-Seidel) update follows from the precomputed cross terms
//    c_ip = sum a_i a_p lambda (k_sv_consts): after pixel i moves by alpha_i, theta1_p changes by
//    -alpha_i c_ip.  The four 1-D solves of a batch are a short scalar recurrence after one warp
//    reduction, instead of four dependent reductions.
//  * Slot records (lengths [g][lane][k] + one offset byte per view group) and batch constants
//    are coalesced register loads, one batch ahead; the band windows are staged with cp.async.
//  * Epilogue: the band's net change e - e0 is folded into global e with red.add (tiles of the
//    same agent that share rows run concurrently), then z, the Mann step and norm partials.
#pragma once
#include "kernels.cuh"

namespace mace {

constexpr int kMaxGroups = 4;  // <= 128 views per agent

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async4(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// shared-memory bytes per warp: the e, lambda and e0 band planes, the state tile with
// halo, and per-pixel v and w
__host__ __device__ constexpr size_t sv_warp_bytes(int S, int ng, int wcap)
{
    return 12 * (size_t)ng * wcap * 32 + 4 * (size_t)((((S + 2) * (S + 2)) + 3) & ~3) + 8 * (size_t)S * S;
}

__device__ __forceinline__ float fast_exp2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// qGGMRF neighbour term with the shared subexpressions fused (icd.py:45-64):
// c = w rho'(d)/d (surrogate coefficient), g = w rho'(d); MUFU log2/exp2.
template <bool kP2>
__device__ __forceinline__ void qg_term(float d, float wk, const PriorC& P, float& g, float& c)
{
    const float ad = fabsf(d);
    if (kP2) {
        // p = 2: rho'(d) = d k(|d|), rho'(d)/d = k(|d|), k = sx^-2 um (q/2 + um) / (1 + um)^2
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

// one batch of slot records in registers: lengths a[p][g][k], offset words, batch constants
// (theta2 x4 | c01 c02 c03 c12 | c13 c23 - -)
template <int K, int NG>
struct SvBatch {
    float a[4][NG][K];
    uint32_t ob[4];
    float4 k0, k1, k2;
};

template <int K, int NG>
__device__ __forceinline__ void load_batch(SvBatch<K, NG>& B, const uint32_t* __restrict__ r,
                                           const float* __restrict__ bk, int recw, int lane)
{
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const uint32_t* q = r + p * recw + (g * 32 + lane) * K;
            if constexpr (K == 2) {
                asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
                    : "=f"(B.a[p][g][0]), "=f"(B.a[p][g][1])
                    : "l"(q));
            } else {
                const float4 v = __ldg(reinterpret_cast<const float4*>(q));
                B.a[p][g][0] = v.x;
                B.a[p][g][1] = v.y;
                B.a[p][g][2] = v.z;
                B.a[p][g][3] = v.w;
            }
        }
        asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(B.ob[p]) : "l"(r + p * recw + NG * 32 * K + lane));
    }
    B.k0 = __ldg(reinterpret_cast<const float4*>(bk));
    B.k1 = __ldg(reinterpret_cast<const float4*>(bk) + 1);
    B.k2 = __ldg(reinterpret_cast<const float4*>(bk) + 2);
}

template <int S, int K, int NG>
__global__ void __launch_bounds__(32, 12) k_icd_sv(PassParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    if (P.done && *P.done) return;
    constexpr int SS = S * S, S2 = S + 2, T2 = S2 * S2, T2p = (T2 + 3) & ~3;
    constexpr int H = S / 2, PER_CLASS = H * H, BPC = (PER_CLASS + 3) / 4, NB = 4 * BPC;
    const int lane = threadIdx.x & 31;
    const int W = P.wcap;
    unsigned char* base = smem + (threadIdx.x >> 5) * sv_warp_bytes(S, NG, W);
    float* se = reinterpret_cast<float*>(base);  // band planes, row R = (g W + o) 32 + lane
    float* sl = se + NG * W * 32;                 // lambda
    float* se0 = sl + NG * W * 32;                // e at staging time
    float* zt = se0 + NG * W * 32;
    float* svv = zt + T2p;
    float* swo = svv + SS;
    const int n = P.n_side;
    const PriorC& PR = P.pr;
    const bool quad = PR.kind == 0;
    const bool p2 = PR.p_is_2;
    const int kk = lane & 7;  // prior: lane 8p + kk owns neighbour kk of batch pixel p (models.py:50-52)
    const int pp = lane >> 3;
    const int ndr = c_dr[kk], ndc = c_dc[kk];
    const float nwk = c_nw[kk];

    for (;;) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(P.head, 1u);
        item = __shfl_sync(FULL, item, 0);
        if (item >= (unsigned)P.n_items) break;
        const uint32_t code = __ldg(P.queue + item);
        const AgentDev& A = P.agents[code >> kAgentShift];
        const int sv = (int)(code & kSvMask);
        float* __restrict__ eg = A.e;
        float* __restrict__ z = A.z;
        float* __restrict__ w = A.w;
        const int V = A.V, recw = A.rec_words;
        constexpr int ng = NG;  // dispatch guarantees A.ng == NG
        const int nsv = A.n_sv_side;
        const int r0 = (sv / nsv) * S, c0 = (sv % nsv) * S;
        const float beta = A.beta_eff, inv_s2 = A.inv_s2;
        const int clamp = A.clamp;
        const uint32_t* __restrict__ recs = A.rec + (size_t)sv * NB * 4 * recw;
        const float* __restrict__ bcs = A.bc + (size_t)sv * NB * 16;

        // -- 1. band windows of this lane's views -> its own bank (cp.async; zero past the window)
        int2 myb[kMaxGroups];
#pragma unroll
        for (int g = 0; g < kMaxGroups; ++g) {
            const int j = 32 * g + lane;
            myb[g] = (g < ng && j < V) ? __ldg(A.band + (size_t)sv * V + j) : make_int2(0, 0);
        }
#pragma unroll
        for (int g = 0; g < kMaxGroups; ++g) {
            if (g >= ng) break;
            const int cnt = myb[g].y;
            const float* ep = eg + myb[g].x;
            const float* lp = A.lam + myb[g].x;
            for (int o = 0; o < W; ++o) {
                const int R = (g * W + o) * 32 + lane;
                if (o < cnt) {
                    cp_async4(se + R, ep + o);
                    cp_async4(sl + R, lp + o);
                    cp_async4(se0 + R, ep + o);
                } else {
                    se[R] = 0.f;
                    sl[R] = 0.f;
                    se0[R] = 0.f;
                }
            }
        }
        cp_async_commit();
        // -- 2. first batch of records
        SvBatch<K, NG> cur, nxt;
        load_batch<K, NG>(cur, recs, bcs, recw, lane);
        // -- 3. tile state + halo, w and v = 2 G(w) - w
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
                if (rr < n && cc < n) {
                    const size_t s = (size_t)rr * n + cc;
                    const float wo = w[s];
                    swo[i] = wo;
                    svv[i] = P.mode ? 2.f * __ldg(P.g + (size_t)A.slice * n * n + s) - wo : A.vt[s];
                } else {
                    svv[i] = 0.f;
                    swo[i] = 0.f;
                }
            }
        }

        // -- 4. batches of four same-parity pixels
        double dsq = 0.0;
        cp_async_wait<0>();  // this lane's band copies have landed
        __syncwarp();        // ... and every other lane's; zt / v / w stores visible
#pragma unroll 1
        for (int b = 0; b < NB; ++b) {
            if (b + 1 < NB) load_batch<K, NG>(nxt, recs + (size_t)(b + 1) * 4 * recw, bcs + (size_t)(b + 1) * 16, recw, lane);
            const float bk[10] = {cur.k0.x, cur.k0.y, cur.k0.z, cur.k0.w, cur.k1.x,
                                  cur.k1.y, cur.k1.z, cur.k1.w, cur.k2.x, cur.k2.y};
            const int cls = b / BPC, ib = (b % BPC) * 4;
            // local pixel of slot p; -1 for padding or off-image slots
            int loc[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int i = ib + p;
                const int lr = (cls >> 1) + 2 * (i / H), lc = (cls & 1) + 2 * (i % H);
                loc[p] = (i < PER_CLASS && r0 + lr < n && c0 + lc < n) ? lr * S + lc : -1;
            }
            // theta1 partials against the band as it stands before the batch
            float num[4];
            int addr[4][NG];
            const auto& av = cur.a;
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int g = 0; g < NG; ++g) addr[p][g] = (g * W + (int)((cur.ob[p] >> (8 * g)) & 0xffu)) * 32 + lane;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) {
                        const float ee = se[addr[p][g] + q * 32], ll = sl[addr[p][g] + q * 32];
                        if (q & 1) a1 = fmaf(av[p][g][q] * ll, ee, a1);
                        else a0 = fmaf(av[p][g][q] * ll, ee, a0);
                    }
                num[p] = a0 + a1;
            }
            // prior of batch pixel pp, neighbour kk (independent across the batch)
            float den_l;
            {
                const int lp = pp == 0 ? loc[0] : pp == 1 ? loc[1] : pp == 2 ? loc[2] : loc[3];
                float g = 0.f, c = 0.f;
                if (lp >= 0 && beta > 0.f) {
                    const int lr = lp / S, lc = lp % S;
                    const int gr = r0 + lr + ndr, gc = c0 + lc + ndc;
                    const bool valid = gr >= 0 && gr < n && gc >= 0 && gc < n;
                    const float wk = valid ? nwk : 0.f;
                    const float d = zt[(lr + 1) * S2 + lc + 1] - zt[(lr + 1 + ndr) * S2 + (lc + 1 + ndc)];
                    if (quad) {
                        g = wk * d;
                        c = wk;
                    } else if (p2) {
                        qg_term<true>(d, wk, PR, g, c);
                    } else {
                        qg_term<false>(d, wk, PR, g, c);
                    }
                }
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    if (pp == p) num[p] -= beta * g;
                den_l = beta * c;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int p = 0; p < 4; ++p) num[p] += __shfl_xor_sync(FULL, num[p], o);
#pragma unroll
            for (int o = 4; o; o >>= 1) den_l += __shfl_xor_sync(FULL, den_l, o);
            float alpha[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float den_p = __shfl_sync(FULL, den_l, 8 * p);
                const int k = loc[p];
                const float zs = k >= 0 ? zt[(k / S + 1) * S2 + k % S + 1] : 0.f;
                float nm = num[p], dn = den_p + bk[p] + inv_s2;
                // coupling to the earlier pixels of the batch (exact Gauss-Seidel order)
                if (p >= 1) nm -= alpha[0] * bk[4 + p - 1];   // c01, c02, c03
                if (p >= 2) nm -= alpha[1] * bk[7 + p - 2];   // c12, c13
                if (p >= 3) nm -= alpha[2] * bk[9];           // c23
                if (quad && beta > 0.f) {
                    nm -= beta * PR.eps2 * zs;
                    dn += beta * PR.eps2;
                }
                nm -= inv_s2 * (zs - (k >= 0 ? svv[k] : 0.f));
                // 1-D solve (icd.py:128-134); the reference skips pixels with den <= 0
                float al = (k >= 0 && dn > 0.f) ? __fdividef(nm, dn) : 0.f;
                if (clamp && zs + al < 0.f) al = -zs;
                alpha[p] = al;
                if (k >= 0 && lane == p) zt[(k / S + 1) * S2 + k % S + 1] = zs + al;
                dsq += (double)al * al;
            }
            // scatter e -= alpha_p a_p in pixel order (a row may be shared within the batch, never
            // within one pixel: load a pixel's rows, then store them)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float ev[NG][K];
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) ev[g][q] = se[addr[p][g] + q * 32];
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) se[addr[p][g] + q * 32] = fmaf(-alpha[p], av[p][g][q], ev[g][q]);
            }
            __syncwarp();  // zt updates visible to the next batch's prior lanes
            cur = nxt;
        }

        // -- 5. fold the band's net change into global e; write z, Mann, partial norms
#pragma unroll
        for (int g = 0; g < kMaxGroups; ++g) {
            if (g >= ng) break;
            const int cnt = myb[g].y;
            float* ep = eg + myb[g].x;
            for (int o = 0; o < cnt; ++o) {
                const int R = (g * W + o) * 32 + lane;
                const float dv = se[R] - se0[R];
                if (dv != 0.f) atomicAdd(ep + o, dv);
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
        if (lane == 0) {  // dsq: every lane holds the same sum (alpha is warp-uniform)
            double* o = P.part + (size_t)item * 4;
            o[0] = dsq;
            o[1] = dw2;
            o[2] = wn2;
            o[3] = wo2;
        }
        __syncwarp();
    }
}

}  // namespace mace
