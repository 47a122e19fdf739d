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
//  * Weighted records (kW, single-slice contexts with lambda > 0): the slot records hold
//    a sqrt(lambda) and the error sinogram is kept as sqrt(lambda) e, so theta1 = sum a lambda e
//    is a plain dot product and the scatter keeps its form (e' -= alpha a'); the band loses its
//    lambda plane (two planes, 2/3 of the shared memory) and each gather is one load.
//  * Pixels are visited in batches of four pixels of one parity class (internal.h): they are
//    never 8-neighbours, so the four prior terms are computed at once on lanes 8p..8p+7, and the
//    data terms theta1_p = sum a_p lambda e are gathered against the band as it stood before the
//    batch.  The exact sequential (Gauss-Seidel) update follows from the precomputed cross terms
//    c_ip = sum a_i a_p lambda (k_sv_consts): after pixel i moves by alpha_i, theta1_p changes by
//    -alpha_i c_ip.  The four 1-D solves of a batch are a short scalar recurrence after one warp
//    reduction, instead of four dependent reductions.
//  * Slot records (per batch one lane-major block: lengths [g][lane][slot][k], offsets [lane][slot]
//    with one byte per view group; internal.h) and batch constants
//    are coalesced register loads, one batch ahead; the band windows are staged with cp.async.
//  * Epilogue: the band's net change e - e0 is folded into global e with red.add (tiles of the
//    same agent that share rows run concurrently), then z, the Mann step and norm partials.
#pragma once
#include <type_traits>
#include "dev_common.cuh"
#include "k2_launch.h"

namespace mace {


__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__host__ __device__ constexpr int sv_rec_words(int ng, int K) { return ng * 32 * K + 32; }

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

// one batch of slot records in registers: lengths a[p][g][k] and offset words
template <int K, int NG>
struct SvBatch {
    float a[4][NG][K];
    uint32_t ob[4];
};

// Visit order of an S x S tile (internal.h sv_slot_pixel): per batch, the local pixel index of each
// of the four slots as a byte (0xff: padding slot); a constant-memory table per tile side.
template <int S>
struct SvOrder {
    struct Table {
        uint32_t v[64];
    };
    static constexpr Table make()
    {
        Table t{};
        constexpr int H = S / 2, PC = H * H, BPC = (PC + 3) / 4;
        for (int b = 0; b < 4 * BPC; ++b) {
            uint32_t w = 0;
            for (int p = 0; p < 4; ++p) {
                const int cls = b / BPC, i = (b % BPC) * 4 + p;
                const uint32_t k = i < PC ? (uint32_t)(((cls >> 1) + 2 * (i / H)) * S + (cls & 1) + 2 * (i % H)) : 0xffu;
                w |= k << (8 * p);
            }
            t.v[b] = w;
        }
        return t;
    }
};
template <int S>
__constant__ typename SvOrder<S>::Table c_svorder = SvOrder<S>::make();

template <int K, int NG>
__device__ __forceinline__ void load_batch(SvBatch<K, NG>& B, const uint32_t* __restrict__ r, int lane)
{
#if !MACE_SV_LANE_MAJOR  // slot-major blocks: per (slot, group) one 8- or 16-byte load, per slot one offset word
    constexpr int RECW = sv_rec_words(NG, K);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const uint32_t* q = r + p * RECW + (g * 32 + lane) * K;
            if constexpr (K == 2) {
                asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(B.a[p][g][0]), "=f"(B.a[p][g][1]) : "l"(q));
            } else {
                asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                    : "=f"(B.a[p][g][0]), "=f"(B.a[p][g][1]), "=f"(B.a[p][g][2]), "=f"(B.a[p][g][3])
                    : "l"(q));
            }
        }
        asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(B.ob[p]) : "l"(r + p * RECW + NG * 32 * K + lane));
    }
    return;
#endif
    // one (batch, chunk) block of records, lane-major (internal.h sv_len_word / sv_ofs_word): the
    // lane's 4 K lengths of a view group are contiguous (one 256-bit load for K = 2, two for K = 4)
    // and its four offset words one 128-bit load
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        const uint32_t* q = r + ((size_t)g * 32 + lane) * 4 * K;
#pragma unroll
        for (int h = 0; h < K / 2; ++h) {  // elements 8h .. 8h + 7 of the lane's [slot][k] run
            float r8[8];
            asm("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(r8[0]), "=f"(r8[1]), "=f"(r8[2]), "=f"(r8[3]), "=f"(r8[4]), "=f"(r8[5]), "=f"(r8[6]),
                  "=f"(r8[7])
                : "l"(q + 8 * h));
#pragma unroll
            for (int i = 0; i < 8; ++i) B.a[(8 * h + i) / K][g][i % K] = r8[i];
        }
    }
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(B.ob[0]), "=r"(B.ob[1]), "=r"(B.ob[2]), "=r"(B.ob[3])
        : "l"(r + (size_t)NG * 32 * 4 * K + 4 * lane));
}

#ifndef MACE_K2_PF
#define MACE_K2_PF 2  // L2 bulk prefetch distance of the slot records in batches (0: off); DESIGN.md §6
#endif
#ifndef MACE_K2_BCPF
#define MACE_K2_BCPF 1  // L2 bulk prefetch of the next tile's batch constants
#endif
#ifndef MACE_K2_NORELOAD
// 1: scatter from registers, the rows an earlier batch pixel shares picked by selects (no band
// reloads: -18 of ~108 shared wavefronts per batch).  Measured slower on B200 (c1 0.536 vs 0.436 ms,
// c2 4.41 vs 3.60 ms; 168 registers): the ~160 extra selects / FMAs per batch cost more issue slots
// than the reloads cost LSU slots.  Kept as an A/B variant; off by default.
#define MACE_K2_NORELOAD 0
#endif
#ifndef MACE_K2_LEAN
// 1: pixel 0 of a batch is scattered by reload-modify-store like the others (6 fewer live registers;
// an occupancy experiment for 16 resident warps per SM)
#define MACE_K2_LEAN 0
#endif
#ifndef MACE_K2_TRIM
// 1: issue trims of the batch step: the qGGMRF p = 2 / no-clamp path as its own loop copy (no
// per-batch tests of the prior kind and the clamp), the zt store index computed by the storing lane
// only, the L2 prefetch pointer advanced per batch, and band addresses by one byte permute
#define MACE_K2_TRIM 1
#endif
#ifndef MACE_K2_BC8
#define MACE_K2_BC8 1  // batch constants by one 256-bit + one 64-bit load (3 loads before)
#endif
#ifndef MACE_K2_V8
#define MACE_K2_V8 1  // 256-bit e-window loads
#endif
#ifndef MACE_K2_MINB
#define MACE_K2_MINB 12  // resident warps per SM the register budget is sized for
#endif
#ifndef MACE_K2_MINB_W
#define MACE_K2_MINB_W 12  // weighted records (16 fits the shared memory but spills registers: slower)
#endif
// MW > 0: multi-warp tiles for agents with more than 128 views (the centralized ICD of
// icd_map_solve, icd.py:306-345, or few agents): warp w of a block owns view chunk w (3 groups of
// 32 views, layout.cpp) of the same tile; per batch the warps exchange their theta1 partials
// through shared memory (one named barrier) and then run identical solves, so every warp's copy
// of the tile state stays identical; warp 0 writes z, w and the norm partials.  MW = 1: up to 8
// chunks per tile, MW = 2: up to kSvMaxChunks.
template <int S, int K, int NG, bool kW, int MW = 0>
__global__ void __launch_bounds__(MW == 0 ? 32 : (MW == 1 ? 256 : 512),
                                  MW == 0 ? (kW ? MACE_K2_MINB_W : MACE_K2_MINB) : 1) k_icd_sv(PassParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    if (P.done && *P.done) return;
    constexpr int SS = S * S, S2 = S + 2, T2 = S2 * S2, T2p = (T2 + 3) & ~3;
    constexpr int H = S / 2, PER_CLASS = H * H, BPC = (PER_CLASS + 3) / 4, NB = 4 * BPC;
    constexpr int RECW = sv_rec_words(NG, K);
    constexpr int U = sv_unit_words(kW);  // words per band row unit: e | lambda [| e0] (kW: e [| e0])
    [[maybe_unused]] constexpr int E0 = U - 32;  // e0 plane offset (MACE_K2_RAW 0)
    const int lane = threadIdx.x & 31;
    const int W = P.wcap;
    const int wid = MW ? (int)(threadIdx.x >> 5) : 0;  // chunk of this warp
    const int CH = MW ? P.chunks : 1;
    unsigned char* base = smem + wid * sv_warp_bytes(S, NG, W, kW);
    // multi-warp tiles: block area after the warps' regions (sv_block_extra_bytes): the next item,
    // warp 0's tile-state snapshot, and the theta1 partials [2][4][CH]
    unsigned* s_item = reinterpret_cast<unsigned*>(smem + CH * sv_warp_bytes(S, NG, W, kW));
    float* s_stage = reinterpret_cast<float*>(s_item + 4);
    float* s_part = s_stage + ((((S + 2) * (S + 2)) + 3) & ~3) + 2 * S * S;
    auto bar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(32 * CH) : "memory"); };
    float* sb = reinterpret_cast<float*>(base);  // band: e at U u + lane, lambda +32[, e0 +E0]
    float* zt = sb + NG * W * U;
    float* svv = zt + T2p;
    float* swo = svv + SS;
    float4* sred = reinterpret_cast<float4*>(swo + SS);  // the batch's {theta1', den, z, v} per pixel, broadcast through smem
#if MACE_K2_RAW
    const int RQ = sv_raw_quads(W);             // 16-byte quads per (group, lane) raw slot
    float4* raw = sred + 4;                     // [g][lane][RQ]: the aligned span of each window
#endif
    const int n = P.n_side;
    const PriorC& PR = P.pr;
    const bool quad_ = PR.kind == 0;
    const bool p2_ = PR.p_is_2;
    const int kk = lane & 7;  // prior: lane 8p + kk owns neighbour kk of batch pixel p (models.py:50-52)
    const int pp = lane >> 3;
    const int ndr = c_dr[kk], ndc = c_dc[kk];
    const float nwk = c_nw[kk];
    const int nofs = ndr * S2 + ndc;

    // work items are pipelined one ahead: the next item's index and code are in flight during the
    // current tile
    // float4 loads per group: a window of a parallel-beam tile spans about S sqrt 2 + 2 channels at
    // channel pitch = pixel pitch, plus up to 3 rows of alignment; wider windows take the slow path
    // VW floats per window load: 8 = one 256-bit load per lane (LDG.256, 32-byte aligned spans: each
    // instruction still touches 32 lines, one per lane's view, so fewer loads = fewer L1 wavefronts)
    constexpr int VW = MACE_K2_V8 ? 8 : 4;
    constexpr int EV = MACE_K2_V8 ? (S * 1414 / 1000 + 16) / 8 : (S * 1414 / 1000 + 8) / 4;
    auto fetch_item = [&]() {
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(P.head, 1u);
        return __shfl_sync(FULL, it, 0);
    };
    auto band_of = [&](uint32_t cd, int2 (&mb)[NG]) {
        const AgentDev& An = P.agents[cd >> kAgentShift];
        const int svn = (int)(cd & kSvMask), Vn = An.V;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int j = 32 * (wid * NG + g) + lane;
            mb[g] = j < Vn ? __ldg(An.band + (size_t)svn * Vn + j) : make_int2(0, 0);
        }
    };
#if MACE_K2_RAW
    // e windows into the raw area: the aligned span of view 32 g + 8 k + (lane & 7) is copied by the
    // four lanes 8 m + (lane & 7), quad v by lane m = v mod 4: one cp.async instruction covers 8
    // views (8 lines) instead of 32, and needs no registers until the owner transposes it
    auto issue_windows = [&](uint32_t cd, const int2 (&mb)[NG]) {
        const float* en = P.agents[cd >> kAgentShift].e;
        const int m = lane >> 3, vl = lane & 7;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int src = 8 * k + vl;
                const int st = __shfl_sync(FULL, mb[g].x, src), cnt = __shfl_sync(FULL, mb[g].y, src);
                const int s0 = st & 3, nv = (cnt + s0 + 3) >> 2;
                float4* dst = raw + (32 * g + src) * RQ + m;
                const float* sp = en + (st - s0) + 4 * m;
                if (m < nv) cp_async16(dst, sp);
                if (m + 4 < nv) cp_async16(dst + 4, sp + 16);
                for (int v = m + 8; v < nv; v += 4) cp_async16(raw + (32 * g + src) * RQ + v, en + (st - s0) + 4 * v);
            }
        cp_async_commit();
    };
#endif
    // e windows: 16-byte loads over the aligned span of each window (a lane's window is one
    // contiguous run of rows; the loads of one instruction hit 32 different lines)
    auto ewin_of = [&](uint32_t cd, const int2 (&mb)[NG], float (&ev)[NG][EV * VW], int (&shf)[NG]) {
        const float* en = P.agents[cd >> kAgentShift].e;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int st = mb[g].x, cnt = mb[g].y;
            shf[g] = st & (VW - 1);
            const float* ep = en + (st - shf[g]);
            const int nv = (cnt + shf[g] + VW - 1) / VW;
#pragma unroll
            for (int v = 0; v < EV; ++v) {
                float* r = ev[g] + VW * v;
                if constexpr (VW == 8) {
                    if (v < nv) {
                        asm volatile("ld.global.cg.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                                       "=f"(r[6]), "=f"(r[7])
                                     : "l"(ep + 8 * v));
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) r[i] = 0.f;
                    }
                } else {
                    const float4 q = v < nv ? __ldcg(reinterpret_cast<const float4*>(ep) + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                    r[0] = q.x;
                    r[1] = q.y;
                    r[2] = q.z;
                    r[3] = q.w;
                }
            }
        }
    };
    // tile state (z with its halo, w, and v = 2 G(w) - w or the explicit target), one tile ahead:
    // loaded after the previous tile's write-back, like the e windows
    constexpr int ZN = (T2 + 31) / 32, VN = (SS + 31) / 32;
    auto state_of = [&](uint32_t cd, float (&zp)[ZN], float (&wp)[VN], float (&vp)[VN]) {
        const AgentDev& An = P.agents[cd >> kAgentShift];
        const int svn = (int)(cd & kSvMask), nsn = An.n_sv_side;
        const int rn = (svn / nsn) * S, cn = (svn % nsn) * S;
        const float* zn = An.z;
#pragma unroll
        for (int k = 0; k < ZN; ++k) {
            const int i = 32 * k + lane;
            const int rr = rn - 1 + i / S2, cc = cn - 1 + i % S2;
            zp[k] = (i < T2 && rr >= 0 && rr < n && cc >= 0 && cc < n) ? __ldcg(zn + (size_t)rr * n + cc) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < VN; ++k) {
            const int i = 32 * k + lane;
            const int rr = rn + i / S, cc = cn + i % S;
            wp[k] = 0.f;
            vp[k] = 0.f;
            if (i < SS && rr < n && cc < n) {
                const size_t s = (size_t)rr * n + cc;
                wp[k] = __ldcg(An.w + s);
                vp[k] = P.mode ? 2.f * __ldg(P.g + (size_t)An.slice * n * n + s) - wp[k] : __ldg(An.vt + s);
            }
        }
    };
    unsigned item;
    if constexpr (MW > 0) {
        if (threadIdx.x == 0) s_item[0] = atomicAdd(P.head, 1u);
        bar();
        item = s_item[0];
    } else {
        item = fetch_item();
    }
    if (item >= (unsigned)P.n_items) return;
    uint32_t code = __ldg(P.queue + item);
    int2 myb[NG];
#if MACE_K2_RAW
    float zpre[ZN], wpre[VN], vpre[VN];
    band_of(code, myb);
    issue_windows(code, myb);
#else
    float ew[NG][EV * VW];
    int sh[NG];
    float zpre[ZN], wpre[VN], vpre[VN];
    band_of(code, myb);
    ewin_of(code, myb, ew, sh);
#endif
    if (!MW || wid == 0) state_of(code, zpre, wpre, vpre);
    int tpar = 1;  // multi-warp: s_item slot of the next item

    for (;;) {
        const AgentDev& A = P.agents[code >> kAgentShift];
        const int sv = (int)(code & kSvMask);
        float* __restrict__ eg = A.e;
        float* __restrict__ z = A.z;
        float* __restrict__ w = A.w;
        const int nsv = A.n_sv_side;
        const int r0 = (sv / nsv) * S, c0 = (sv % nsv) * S;
        const bool full = r0 + S <= n && c0 + S <= n;  // interior tile: no image-edge checks
        const float beta = A.beta_eff, inv_s2 = A.inv_s2;
        const int clamp_ = A.clamp;
        // records [sv][batch][chunk][slot][RECW]: this warp's chunk, batch stride BST
        const size_t BST = (size_t)CH * 4 * RECW;
        const uint32_t* __restrict__ recs = A.rec + (size_t)sv * NB * BST + (size_t)wid * 4 * RECW;
        const float* __restrict__ bcs = A.bc + (size_t)sv * NB * 16;
        // next item
        unsigned nitem;
        if constexpr (MW > 0) {
            // warp 0 fetches the next item and publishes its snapshot of this tile's state; one
            // barrier, then every warp starts from the same state
            if (threadIdx.x == 0) s_item[tpar] = atomicAdd(P.head, 1u);
            if (wid == 0) {
#pragma unroll
                for (int k = 0; k < ZN; ++k)
                    if (32 * k + lane < T2) s_stage[32 * k + lane] = zpre[k];
#pragma unroll
                for (int k = 0; k < VN; ++k)
                    if (32 * k + lane < SS) {
                        s_stage[T2p + 32 * k + lane] = wpre[k];
                        s_stage[T2p + SS + 32 * k + lane] = vpre[k];
                    }
            }
            bar();
            nitem = s_item[tpar];
            tpar ^= 1;
#pragma unroll
            for (int k = 0; k < ZN; ++k)
                if (32 * k + lane < T2) zpre[k] = s_stage[32 * k + lane];
#pragma unroll
            for (int k = 0; k < VN; ++k)
                if (32 * k + lane < SS) {
                    wpre[k] = s_stage[T2p + 32 * k + lane];
                    vpre[k] = s_stage[T2p + SS + 32 * k + lane];
                }
        } else {
            nitem = fetch_item();
        }
        const bool more = nitem < (unsigned)P.n_items;
        const uint32_t ncode = more ? __ldg(P.queue + nitem) : 0u;
#if MACE_K2_PF > 0
        // the next tile's records, for the L2 prefetch that runs MACE_K2_PF batches ahead
        const uint32_t* nrecs = more ? P.agents[ncode >> kAgentShift].rec + (size_t)(ncode & kSvMask) * NB * BST +
                                           (size_t)wid * 4 * RECW
                                     : nullptr;
#endif
#if MACE_K2_BCPF
        // the next tile's batch constants (1 KB, read from the first batch on) into L2 a whole tile
        // ahead: at config 2 they do not stay in L2 between passes (16 agents x 16.8 MB)
        if (lane == 0 && wid == 0 && more)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.agents[ncode >> kAgentShift].bc +
                                                                            (size_t)(ncode & kSvMask) * NB * 16),
                         "r"((uint32_t)(NB * 16 * 4))
                         : "memory");
#endif

        // -- 1. band: lambda rows by one coalesced copy, e rows from the prefetched windows
        if constexpr (!kW) {  // lambda: pre-arranged per tile (k_sv_consts) as [u][32]; 16-byte copies into the units
            const float* lsrc = A.lb + ((size_t)sv * CH + wid) * NG * W * 32;
            for (int c = lane; c < NG * W * 8; c += 32) cp_async16(sb + (c >> 3) * U + 32 + 4 * (c & 7), lsrc + 4 * c);
            cp_async_commit();
        }
        // -- 2. first batch of records
        SvBatch<K, NG> cur, nxt;
        load_batch<K, NG>(cur, recs, lane);
        // batch constants (theta2 x4 | c01 c02 c03 c12 | c13 c23 - -), 1 KB per tile: into L1 now,
        // read per batch as broadcast loads
        if (lane < NB / 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(bcs + 32 * lane));
        // -- 3. tile state + halo, w and v = 2 G(w) - w (prefetched)
#pragma unroll
        for (int k = 0; k < ZN; ++k)
            if (32 * k + lane < T2) zt[32 * k + lane] = zpre[k];
#pragma unroll
        for (int k = 0; k < VN; ++k)
            if (32 * k + lane < SS) {
                swo[32 * k + lane] = wpre[k];
                svv[32 * k + lane] = vpre[k];
            }

        // -- 4. batches of four same-parity pixels
        float dsq = 0.f;
#if MACE_K2_RAW
        // e plane from the raw windows (rows past the window are zero); the raw slot is this lane's
        // own view, read as 16-byte quads (conflict-free: RQ is odd)
        if constexpr (kW) cp_async_wait<0>();
        else cp_async_wait<1>();  // the window group (committed last tile), not this tile's lambda copies
        __syncwarp();
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int cnt = myb[g].y, s0 = myb[g].x & 3;
            float* d = sb + g * W * U + lane;
            const float4* rr = raw + (size_t)(32 * g + lane) * RQ;
#pragma unroll 2
            for (int v = 0; v < RQ; ++v) {
                const float4 x4 = rr[v];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int o = 4 * v + i - s0;
                    if (o >= 0 && o < W) {
                        const float xi = i == 0 ? x4.x : i == 1 ? x4.y : i == 2 ? x4.z : x4.w;
                        d[o * U] = o < cnt ? xi : 0.f;
                    }
                }
            }
        }
#else
        // e and e0 planes from the registers (rows past the window are zero)
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int cnt = myb[g].y;
            float* d = sb + g * W * U + lane;
            if (W <= VW * EV - (VW - 1)) {
#pragma unroll
                for (int v = 0; v < EV * VW; ++v) {
                    {
                        const int o = v - sh[g];
                        if (o >= 0 && o < W) {
                            const float x = o < cnt ? ew[g][v] : 0.f;
                            d[o * U] = x;
                            d[o * U + E0] = x;
                        }
                    }
                }
            } else {  // wide windows: plain row loads
                for (int o = 0; o < W; ++o) {
                    const float x = o < cnt ? __ldcg(eg + myb[g].x + o) : 0.f;
                    d[o * U] = x;
                    d[o * U + E0] = x;
                }
            }
        }
#endif
        if constexpr (!kW) cp_async_wait<0>();  // this lane's lambda copies have landed
        __syncwarp();        // ... and every other lane's; band / zt / v / w stores visible
        // kFull: the tile lies inside the image (all but the last tile row / column), so no slot
        // needs the image-edge test
#if MACE_K2_PF > 0 && MACE_K2_TRIM
        // L2 prefetch pointer of batch b + PF: this tile's records, then the next tile's
        const uint32_t* pfp = MACE_K2_PF < NB ? recs + (size_t)MACE_K2_PF * BST : nrecs;
#endif
        // kFast: qGGMRF with p = 2 (the fused qg_term), no quadratic term, no clamp -- the configured
        // path of every benchmark -- compiled without the per-batch tests
        auto step = [&](const int b, const SvBatch<K, NG>& C, SvBatch<K, NG>& Nx, auto full_tag, auto fast_tag) {
            constexpr bool kFull = decltype(full_tag)::value;
            constexpr bool kFast = decltype(fast_tag)::value;
            const bool quad = kFast ? false : quad_;
            const bool p2 = kFast ? true : p2_;
            const int clamp = kFast ? 0 : clamp_;
            if (b + 1 < NB) load_batch<K, NG>(Nx, recs + (size_t)(b + 1) * BST, lane);
#if MACE_K2_PF > 0 && MACE_K2_TRIM
            if (lane == 0 && pfp)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pfp), "r"((uint32_t)(4 * RECW * 4))
                             : "memory");
            pfp = b + MACE_K2_PF + 1 == NB ? nrecs : (pfp ? pfp + BST : nullptr);
#elif MACE_K2_PF > 0
            // records of batch b + PF (this tile's or the next one's) pulled into L2 by one bulk
            // prefetch (TMA unit, no LSU work, no registers): the register load one batch ahead then
            // sees L2 rather than DRAM latency
            if (lane == 0) {
                const int tb = b + MACE_K2_PF;
                const uint32_t* pf = tb < NB ? recs + (size_t)tb * BST
                                             : (nrecs ? nrecs + (size_t)(tb - NB) * BST : nullptr);
                if (pf)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"((uint32_t)(4 * RECW * 4))
                                 : "memory");
            }
#endif
#if MACE_K2_BC8  // the batch's theta2 x4 and first four cross terms as one 256-bit broadcast load
            float bk[10];
            asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(bk[0]), "=f"(bk[1]), "=f"(bk[2]), "=f"(bk[3]), "=f"(bk[4]), "=f"(bk[5]), "=f"(bk[6]), "=f"(bk[7])
                : "l"(bcs + 16 * b));
            {
                const float2 k2 = __ldg(reinterpret_cast<const float2*>(bcs + 16 * b + 8));
                bk[8] = k2.x;
                bk[9] = k2.y;
            }
#else
            const float4 k0 = __ldg(reinterpret_cast<const float4*>(bcs + 16 * b));
            const float4 k1 = __ldg(reinterpret_cast<const float4*>(bcs + 16 * b) + 1);
            const float2 k2 = __ldg(reinterpret_cast<const float2*>(bcs + 16 * b + 8));
            const float bk[10] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w, k2.x, k2.y};
#endif
            // local pixel kx = lr S + lc of slot p (visit-order table); ok = real and inside the image
            const uint32_t kxw = c_svorder<S>.v[b];
            int kx[4];
            bool ok[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                kx[p] = (int)((kxw >> (8 * p)) & 0xffu);
                ok[p] = (PER_CLASS % 4 == 0 || kx[p] != 0xff) &&
                        (kFull || (r0 + kx[p] / S < n && c0 + kx[p] % S < n));
                if (PER_CLASS % 4 != 0 && kx[p] == 0xff) kx[p] = 0;
            }
            // theta1 partials against the band as it stands before the batch
            float num[4];
#if MACE_K2_NORELOAD
            float gv[4][NG][K];  // every pixel's rows as gathered (before the batch touched them)
#elif !MACE_K2_LEAN
            float e0v[NG][K];  // pixel 0's rows as gathered (nothing in the batch has touched them yet)
#endif
            int ab[4][NG];  // byte offsets of the slots' first rows in the band
            const auto& av = C.a;
#define BANDB(a, q, plane) (*reinterpret_cast<float*>(reinterpret_cast<char*>(sb) + (a) + 4 * ((q) * U + (plane))))
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if constexpr (MACE_K2_TRIM && U == 64)  // 4 o U bytes = byte g of the offset word moved to bits 8..15
                        ab[p][g] = (int)__byte_perm(C.ob[p], 0u, 0x4404u | (g << 4)) + 4 * (g * W * U + lane);
                    else
                        ab[p][g] = 4 * ((g * W + (int)((C.ob[p] >> (8 * g)) & 0xffu)) * U + lane);
                }
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) {
                        const float ee = BANDB(ab[p][g], q, 0);
#if MACE_K2_NORELOAD
                        gv[p][g][q] = ee;
#elif !MACE_K2_LEAN
                        if (p == 0) e0v[g][q] = ee;
#endif
                        // kW: a' = a sqrt(lambda) against e' = sqrt(lambda) e
                        const float al = kW ? av[p][g][q] : av[p][g][q] * BANDB(ab[p][g], q, 32);
                        if (q & 1) a1 = fmaf(al, ee, a1);
                        else a0 = fmaf(al, ee, a0);
                    }
                num[p] = a0 + a1;
            }
            // prior of batch pixel pp, neighbour kk (independent across the batch)
            float den_l, den4[4], zs4[4], vv4[4];
            {
                int kl = (int)((kxw >> (8 * pp)) & 0xffu);
                const bool okl = (PER_CLASS % 4 == 0 || kl != 0xff) && (kFull || (r0 + kl / S < n && c0 + kl % S < n));
                if (PER_CLASS % 4 != 0 && kl == 0xff) kl = 0;
                // z and v of this lane's batch pixel (the group leader passes them on)
                const float zlead = zt[(kl / S + 1) * S2 + kl % S + 1], vlead = svv[kl];
                float g = 0.f, c = 0.f;
                if (okl && beta > 0.f) {
                    const int lr = kl / S, lc = kl % S;
                    const int gr = r0 + lr + ndr, gc = c0 + lc + ndc;
                    const bool valid = gr >= 0 && gr < n && gc >= 0 && gc < n;
                    const float wk = valid ? nwk : 0.f;
                    const int ci = (lr + 1) * S2 + lc + 1;
                    const float d = zt[ci] - zt[ci + nofs];
                    if (quad) {
                        g = wk * d;
                        c = wk;
                    } else if (p2) {
                        qg_term<true>(d, wk, PR, g, c);
                    } else {
                        qg_term<false>(d, wk, PR, g, c);
                    }
                }
                den_l = beta * c;
                // theta1 of the four pixels by a splitting butterfly: after the xor-16 and xor-8
                // stages lanes 8p..8p+7 hold partial sums of pixel p = lane >> 3 only (the pixel
                // whose prior neighbour they own), which the xor-4/2/1 stages finish with the
                // prior gradient folded in: 6 shuffles instead of 20
                const bool h16 = lane & 16, h8 = lane & 8;
                float k0 = h16 ? num[2] : num[0], k1 = h16 ? num[3] : num[1];
                k0 += __shfl_xor_sync(FULL, h16 ? num[0] : num[2], 16);
                k1 += __shfl_xor_sync(FULL, h16 ? num[1] : num[3], 16);
                float kp = h8 ? k1 : k0;
                kp += __shfl_xor_sync(FULL, h8 ? k0 : k1, 8);
                if (!MW || wid == 0) kp -= beta * g;  // the prior gradient once per block
#pragma unroll
                for (int o = 4; o; o >>= 1) {
                    kp += __shfl_xor_sync(FULL, kp, o);
                    den_l += __shfl_xor_sync(FULL, den_l, o);
                }
                if constexpr (MW > 0) {  // theta1 = sum of the chunks' partials, in chunk order in every warp
                    float* sp = s_part + ((b & 1) * 4 + pp) * CH;
                    if ((lane & 7) == 0) sp[wid] = kp;
                    bar();
                    float t = 0.f;
                    for (int w2 = 0; w2 < CH; ++w2) t += sp[w2];
                    kp = t;
                }
#pragma unroll
                // every lane needs all four pixels' sums and their z, v: the group leaders store
                // {num_p, den_p, z_p, v_p} and every lane reads them back as four broadcast 16-byte loads
                // (7 LSU operations instead of 8 shuffles and 8 scalar loads)
                __syncwarp();  // the previous batch's reads are done
                if ((lane & 7) == 0) sred[pp] = make_float4(kp, den_l, zlead, vlead);
                __syncwarp();
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float4 r = sred[p];
                    num[p] = r.x;
                    den4[p] = r.y;
                    zs4[p] = r.z;
                    vv4[p] = r.w;
                }
            }
            // the four 1-D solves (icd.py:128-134): everything but the coupling to earlier pixels of
            // the batch is independent across p; the reference skips pixels with den <= 0
            float nm[4], rd[4], zs[4];
#if !MACE_K2_TRIM
            int ci[4];
#endif
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float den_p = den4[p];
#if !MACE_K2_TRIM
                ci[p] = (kx[p] / S + 1) * S2 + kx[p] % S + 1;
#endif
                zs[p] = zs4[p];
                float dn = den_p + bk[p] + inv_s2;
                nm[p] = num[p];
                if (quad && beta > 0.f) {
                    nm[p] -= beta * PR.eps2 * zs[p];
                    dn += beta * PR.eps2;
                }
                nm[p] -= inv_s2 * (zs[p] - vv4[p]);
                float r;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dn));
                rd[p] = (ok[p] && dn > 0.f) ? r : 0.f;
            }
            // coupling to the earlier pixels of the batch (exact Gauss-Seidel order)
            float alpha[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float al = ok[p] ? nm[p] * rd[p] : 0.f;
                if (clamp && zs[p] + al < 0.f) al = ok[p] ? -zs[p] : 0.f;
                alpha[p] = al;
                if (p == 0) {
                    nm[1] -= al * bk[4];
                    nm[2] -= al * bk[5];
                    nm[3] -= al * bk[6];
                } else if (p == 1) {
                    nm[2] -= al * bk[7];
                    nm[3] -= al * bk[8];
                } else if (p == 2) {
                    nm[3] -= al * bk[9];
                }
                dsq = fmaf(al, al, dsq);
            }
            {  // lane p < 4 stores pixel p's new value (one store instead of four); the next reads of
               // zt by other lanes come after a __syncwarp
                float zn = zs[0] + alpha[0];
                bool okw = ok[0];
#if MACE_K2_TRIM
                const int km = (int)((kxw >> (8 * (lane & 3))) & 0xffu);  // this lane's slot pixel
                const int cw = (km / S + 1) * S2 + km % S + 1;
#else
                int cw = ci[0];
#endif
#pragma unroll
                for (int p = 1; p < 4; ++p)
                    if (lane == p) {
                        zn = zs[p] + alpha[p];
#if !MACE_K2_TRIM
                        cw = ci[p];
#endif
                        okw = ok[p];
                    }
                if (lane < 4 && okw) zt[cw] = zn;
                __syncwarp();
            }
#if MACE_K2_NORELOAD
            // scatter e -= alpha_p a_p in pixel order without reading the band back: pixel p's rows
            // start from their gathered values, take the updates of the earlier batch pixels that
            // share them (row (p, k) == row (q, k') iff the slots' window offsets differ by k' - k,
            // i.e. ab[p] - ab[q] == (k' - k) U; a row is never shared within one pixel), then its
            // own: the same operations in the same order as updating the band pixel by pixel, and
            // the last store to a shared row carries every update
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    float ev[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) ev[k] = gv[p][g][k];
#pragma unroll
                    for (int q = 0; q < p; ++q) {
                        const int d = (ab[p][g] - ab[q][g]) / 4;
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            // the length of q's entry on this row, 0 if q does not touch it (selects, not
                            // branches: the lanes disagree); fmaf(-alpha, 0, e) == e
                            float sel = 0.f;
#pragma unroll
                            for (int k2 = 0; k2 < K; ++k2) sel = d == (k2 - k) * U ? av[q][g][k2] : sel;
                            ev[k] = fmaf(-alpha[q], sel, ev[k]);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) BANDB(ab[p][g], k, 0) = fmaf(-alpha[p], av[p][g][k], ev[k]);
                }
#else
            // scatter e -= alpha_p a_p in pixel order (a row may be shared within the batch, never
            // within one pixel): pixel 0 from the gathered values, then reload-modify-store
#if !MACE_K2_LEAN
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int q = 0; q < K; ++q) BANDB(ab[0][g], q, 0) = fmaf(-alpha[0], av[0][g][q], e0v[g][q]);
#endif
#pragma unroll
            for (int p = MACE_K2_LEAN ? 0 : 1; p < 4; ++p) {
                float ev[NG][K];
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) ev[g][q] = BANDB(ab[p][g], q, 0);
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) BANDB(ab[p][g], q, 0) = fmaf(-alpha[p], av[p][g][q], ev[g][q]);
            }
#endif
        };
        // ping-pong record buffers (NB is a multiple of 4); one loop copy per (full, fast) pair
#define K2_BATCHES(FT, KT)                                 \
    _Pragma("unroll 1") for (int b = 0; b < NB; b += 2)    \
    {                                                      \
        step(b, cur, nxt, FT{}, KT{});                     \
        step(b + 1, nxt, cur, FT{}, KT{});                 \
    }
        const bool fast = MACE_K2_TRIM && !quad_ && p2_ && !clamp_;
        if (fast) {
            if (full) {
                K2_BATCHES(std::true_type, std::true_type)
            } else {
                K2_BATCHES(std::false_type, std::true_type)
            }
        } else {
            if (full) {
                K2_BATCHES(std::true_type, std::false_type)
            } else {
                K2_BATCHES(std::false_type, std::false_type)
            }
        }
#undef K2_BATCHES

        // -- 5. fold the band's net change into global e (vector red.add over the window's aligned
        // 16-byte span: rows outside the window add +0); write z, Mann, partial norms
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int st = myb[g].x, cnt = myb[g].y, s0 = st & 3;
            float* ep = eg + (st - s0);
            const float* d = sb + g * W * U + lane;
            const int nv = (cnt + s0 + 3) >> 2;
#if MACE_K2_RAW
            const float4* rr = raw + (size_t)(32 * g + lane) * RQ;  // the snapshot e0 the band was staged from
#endif
            for (int v = 0; v < nv; ++v) {
                float dv[4];
#if MACE_K2_RAW
                const float4 r4 = rr[v];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int o = 4 * v + i - s0;
                    const float e0 = i == 0 ? r4.x : i == 1 ? r4.y : i == 2 ? r4.z : r4.w;
                    dv[i] = (o >= 0 && o < cnt) ? d[o * U] - e0 : 0.f;
                }
#else
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int o = 4 * v + i - s0;
                    dv[i] = (o >= 0 && o < cnt) ? d[o * U] - d[o * U + E0] : 0.f;
                }
#endif
                if (P.det) {  // integer adds commute: the class's sum is independent of the tile order
                    unsigned long long* q = A.ed + (st - s0) + 4 * v;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (dv[i] != 0.f)
                            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(q + i),
                                         "l"((unsigned long long)__double2ll_rn((double)dv[i] * kDetScale))
                                         : "memory");
                } else if (dv[0] != 0.f || dv[1] != 0.f || dv[2] != 0.f || dv[3] != 0.f)
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ep + 4 * v), "f"(dv[0]),
                                 "f"(dv[1]), "f"(dv[2]), "f"(dv[3])
                                 : "memory");
            }
        }

        double dw2 = 0.0, wn2 = 0.0, wo2 = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < SS; i0 += 32) {
            const int i = i0 + lane;
            const int rr = r0 + i / S, cc = c0 + i % S;
            if (i < SS && rr < n && cc < n && wid == 0) {
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
        if (lane == 0 && wid == 0) {  // dsq: every lane holds the same sum (alpha is warp-uniform)
            double* o = P.part + (size_t)item * 4;
            o[0] = (double)dsq;
            o[1] = dw2;
            o[2] = wn2;
            o[3] = wo2;
        }
        __syncwarp();  // every lane's write-back reads of the band and the raw area are done
        if (!more) break;
        item = nitem;
        code = ncode;
        band_of(code, myb);
#if MACE_K2_RAW
        issue_windows(code, myb);
#else
        ewin_of(code, myb, ew, sh);
#endif
        if (!MW || wid == 0) state_of(code, zpre, wpre, vpre);
    }
}

}  // namespace mace
