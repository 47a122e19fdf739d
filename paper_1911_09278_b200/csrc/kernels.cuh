// Device code for the MACE hot path on sm_100a.
//
//   K2  k_icd_sv / k_icd_raster   one partial-update ICD pass per agent
//                                 (restates _sweep, pkg/src/macetomo/icd.py:67-139,
//                                 with v = 2G(w)-w (mace.py:99-102) fused in front and
//                                 the Mann step (mace.py:111-117) fused behind)
//   K3  k_fp_agents / k_fp_rows   forward projection, e = y - A z (icd.py:200,210-211;
//                                 geometry.py:261-270)
//       k_like / k_prior_cost     costs (models.py:235-257)
//   K4  k_consensus / k_norms /   average (mace.py:71-90), relnorm and divergence test
//       k_finish                  (mace.py:309-318), log row
#pragma once
#include "dev_common.cuh"

namespace mace {

// K2 super-voxel pass: see k_sv.cuh (compiled per tile side in k2_inst.cu).

// ===========================================================================
// K2 raster pass: the reference's exact visiting order (pixels 0..n-1), one
// warp per agent, e and z in global memory.  This is the per-pass parity mode
// (it reproduces partial_update_prox pass by pass, to fp32 rounding).
// ===========================================================================
template <int NV>
__global__ void __launch_bounds__(32) k_icd_raster(PassParams P, int agent_base)
{
    if (P.done && *P.done) return;
    const int lane = threadIdx.x & 31;
    const int item = blockIdx.x;
    const AgentDev& A = P.agents[agent_base + item];
    const int n = P.n_side;
    const PriorC& PR = P.pr;
    float* eg = A.e;
    const float* lam = A.lam;
    float* z = A.z;
    const float beta = A.beta_eff, inv_s2 = A.inv_s2;
    double dsq = 0.0;
    const size_t N = (size_t)n * n;
    for (size_t s = (size_t)P.s_begin; s < (size_t)P.s_end && s < N; ++s) {
        const int2 pe = A.rpix[s];
        const int r = (int)(s / n), col = (int)(s % n);
        const float zs = __ldcg(z + s);
        float vv4[NV][4];
        uint32_t ii4[NV][4];
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int e0 = 4 * (lane + 32 * j);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                vv4[j][q] = 0.f;
                ii4[j][q] = 0;
            }
            if (e0 < pe.y) {
                const float4 v4 = *reinterpret_cast<const float4*>(A.rval + pe.x + e0);
                const uint4 i4 = *reinterpret_cast<const uint4*>(A.ridx + pe.x + e0);
                vv4[j][0] = v4.x; vv4[j][1] = v4.y; vv4[j][2] = v4.z; vv4[j][3] = v4.w;
                ii4[j][0] = i4.x; ii4[j][1] = i4.y; ii4[j][2] = i4.z; ii4[j][3] = i4.w;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (e0 + q < pe.y) {
                    const uint32_t r = ii4[j][q];
                    t = fmaf(vv4[j][q] * __ldg(lam + r), __ldcg(eg + r), t);
                }
        }
        float g, c;
        {
            const int kk = lane & 7;
            const int gr = r + c_dr[kk], gc = col + c_dc[kk];
            const bool valid = gr >= 0 && gr < n && gc >= 0 && gc < n;
            const float zr = valid ? __ldcg(z + (size_t)gr * n + gc) : 0.f;
            prior_lane(lane, zs, zr, valid && beta > 0.f, PR, g, c);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t += __shfl_xor_sync(FULL, t, o);
            g += __shfl_xor_sync(FULL, g, o);
            c += __shfl_xor_sync(FULL, c, o);
        }
        const float v = P.mode ? 2.f * P.g[(size_t)A.slice * N + s] - A.w[s] : A.vt[s];
        float alpha;
        if (pixel_step(t, g, c, zs, v, A.th[s], beta, inv_s2, A.clamp, PR, alpha)) {
            if (lane == 0) {
                __stcg(z + s, zs + alpha);
                dsq += (double)alpha * alpha;
            }
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int e0 = 4 * (lane + 32 * j);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (e0 + q < pe.y) {
                        float* ep = eg + ii4[j][q];
                        __stcg(ep, __ldcg(ep) - alpha * vv4[j][q]);
                    }
            }
        }
        __syncwarp();
    }
    // fused Mann step (mace.py:307) over the whole image
    double dw2 = 0.0, wn2 = 0.0, wo2 = 0.0;
    if (P.mode) {
        for (size_t s = lane; s < N; s += 32) {
            const float zn = __ldcg(z + s);
            const float wo = A.w[s];
            const float v = 2.f * P.g[(size_t)A.slice * N + s] - wo;
            const float wn = P.rho * (2.f * zn - v) + (1.f - P.rho) * wo;
            A.w[s] = wn;
            const double dd = (double)wn - (double)wo;
            dw2 += dd * dd;
            wn2 += (double)wn * wn;
            wo2 += (double)wo * wo;
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
}

// ===========================================================================
// K3: forward projection.  One warp per sinogram row over the global CSR
// (fixed reduction order -> deterministic).  Agent refresh writes
// e = y - A_i z into the agent's interleaved {e, lambda} array.
// ===========================================================================
struct FPParams {
    const int64_t* rp;
    const int* cols;
    const float* vals;
    int n_ch;
};

// sum over one CSR row of vals[k] * x[cols[k]], lanes strided, four independent accumulators
// (loads of four chunks in flight); fixed order -> deterministic
__device__ __forceinline__ float row_dot(const FPParams& F, int64_t k0, int64_t k1, const float* __restrict__ x,
                                        int lane)
{
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int64_t k = k0 + lane;
    for (; k + 96 < k1; k += 128) {
        const int c0 = __ldcs(F.cols + k), c1 = __ldcs(F.cols + k + 32), c2 = __ldcs(F.cols + k + 64),
                  c3 = __ldcs(F.cols + k + 96);
        const float v0 = __ldcs(F.vals + k), v1 = __ldcs(F.vals + k + 32), v2 = __ldcs(F.vals + k + 64),
                    v3 = __ldcs(F.vals + k + 96);
        a0 = fmaf(v0, __ldcg(x + c0), a0);
        a1 = fmaf(v1, __ldcg(x + c1), a1);
        a2 = fmaf(v2, __ldcg(x + c2), a2);
        a3 = fmaf(v3, __ldcg(x + c3), a3);
    }
    for (; k < k1; k += 32) a0 = fmaf(__ldcs(F.vals + k), __ldcg(x + __ldcs(F.cols + k)), a0);
    return warp_sum((a0 + a1) + (a2 + a3));
}

// agent owning concatenated row `wr`: last a with row_base[a] <= wr (row_base ascending)
__device__ __forceinline__ int agent_of_row(const int* row_base, int n_agents, int wr)
{
    int lo = 0, hi = n_agents - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (row_base[mid] <= wr) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void k_fp_agents(FPParams F, const AgentDev* agents, const int* row_base, int n_agents,
                            int total_rows, const int* done)
{
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int wr = gw; wr < total_rows; wr += nw) {
        const int a = agent_of_row(row_base, n_agents, wr);
        const AgentDev& A = agents[a];
        const int r = wr - row_base[a];
        if (r >= A.R) continue;  // alignment padding between agents
        const int j = r / F.n_ch, ch = r % F.n_ch;
        const int64_t g = (int64_t)A.views[j] * F.n_ch + ch;
        const float acc = row_dot(F, F.rp[g], F.rp[g + 1], A.z, lane);
        if (lane == 0) A.e[r] = A.sq ? A.sq[r] * (A.y[r] - acc) : A.y[r] - acc;
    }
}

// out[g] = (A x)[g] for all rows; optional weighted residual partials 0.5 lambda (y - Ax)^2
__global__ void k_fp_rows(FPParams F, int n_rows, const float* x, float* out, const float* y, const float* lam,
                          double* part)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    double loc = 0.0;
    for (int g = gw; g < n_rows; g += nw) {
        const float acc = row_dot(F, F.rp[g], F.rp[g + 1], x, lane);
        if (lane == 0) {
            if (out) out[g] = acc;
            if (part) {
                const double r = (double)y[g] - (double)acc;
                loc += 0.5 * (double)lam[g] * r * r;
            }
        }
    }
    if (part) {
        __shared__ double sh[32];
        if (lane == 0) sh[threadIdx.x >> 5] = loc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
            part[blockIdx.x] = s;
        }
    }
}

// beta * h(x), pairs s < r only (models.py:111-118,248-257), fp64 arithmetic
__device__ __forceinline__ double qg_potential_d(double d, const PriorC& P)
{
    const double ad = fabs(d);
    const double u = ad / (P.T * P.sx);
    if (!(u > 0.0)) return 0.0;
    const double um = pow(u, P.q - P.p);
    return (pow(ad, P.p) / (P.p * pow(P.sx, P.p))) * (um / (1.0 + um));
}

// rho'(d) in fp64 (icd.py:45-64 _qg_influence, reference convention)
__device__ __forceinline__ double qg_influence_d(double d, const PriorC& P)
{
    const double ad = fabs(d);
    const double u = ad / (P.T * P.sx);
    if (!(u > 0.0)) return 0.0;
    const double um = pow(u, P.q - P.p);
    const double g = pow(ad, P.p - 1.0) / pow(P.sx, P.p) * um * (P.q / P.p + um) / ((1.0 + um) * (1.0 + um));
    return d < 0.0 ? -g : g;
}

// MAP-cost gradient, data part: grad[s] -= sum_rows a_rs lambda_r (y_r - (Ax)_r)  (one warp per row)
__global__ void k_bp_rows(FPParams F, int n_rows, const float* Ax, const float* y, const float* lam, double* grad)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int g = gw; g < n_rows; g += nw) {
        const double r = (double)lam[g] * ((double)y[g] - (double)Ax[g]);
        if (r == 0.0) continue;
        for (int64_t k = F.rp[g] + lane; k < F.rp[g + 1]; k += 32) atomicAdd(grad + F.cols[k], -(double)F.vals[k] * r);
    }
}

// back-projection out[s] += sum_rows a_rs sino_r (geometry.py:273-282), one warp per row, fp64 atomics
__global__ void k_bp_sino(FPParams F, int n_rows, const float* sino, double* out)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int g = gw; g < n_rows; g += nw) {
        const double r = (double)sino[g];
        if (r == 0.0) continue;
        for (int64_t k = F.rp[g] + lane; k < F.rp[g + 1]; k += 32) atomicAdd(out + F.cols[k], (double)F.vals[k] * r);
    }
}

// MAP-cost gradient, prior part: grad[s] += beta sum_k w_k rho'(x_s - x_k) (+ 2 beta eps x_s, quadratic)
__global__ void k_prior_grad(const float* x, int n_side, PriorC P, double beta, double* grad)
{
    const size_t N = (size_t)n_side * n_side;
    for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < N; s += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(s / n_side), c = (int)(s % n_side);
        const double xs = x[s];
        double acc = 0.0;
        for (int k = 0; k < 8; ++k) {
            const int rr = r + c_dr[k], cc = c + c_dc[k];
            if (rr < 0 || rr >= n_side || cc < 0 || cc >= n_side) continue;
            const double d = xs - (double)x[(size_t)rr * n_side + cc];
            acc += (double)c_nw[k] * (P.kind == 0 ? d : qg_influence_d(d, P));
        }
        if (P.kind == 0) acc += 2.0 * P.eps * xs;
        grad[s] += beta * acc;
    }
}

__global__ void k_prior_cost(const float* x, int n_side, PriorC P, double* part)
{
    const size_t N = (size_t)n_side * n_side;
    double loc = 0.0;
    for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < N; s += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(s / n_side), c = (int)(s % n_side);
        const double xs = x[s];
        for (int k = 4; k < 8; ++k) {  // offsets (0,1), (1,-1), (1,0), (1,1): exactly the r > s partners
            const int rr = r + c_dr[k], cc = c + c_dc[k];
            if (rr < 0 || rr >= n_side || cc < 0 || cc >= n_side) continue;
            const double d = xs - (double)x[(size_t)rr * n_side + cc];
            const double wk = (double)c_nw[k];
            loc += P.kind == 0 ? 0.5 * wk * d * d : wk * qg_potential_d(d, P);
        }
        if (P.kind == 0) loc += P.eps * xs * xs;
    }
    __shared__ double sh[256];
    sh[threadIdx.x] = loc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// ===========================================================================
// theta2 = sum_rows a^2 lambda per pixel (icd.py:193-195), deterministic
// ===========================================================================
__global__ void k_theta2_raster(const AgentDev* agents, int n_agents, int n)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const long total = (long)n_agents * n;
    for (long it = gw; it < total; it += nw) {
        const AgentDev& A = agents[it / n];
        const int s = (int)(it % n);
        const int2 pe = A.rpix[s];
        float acc = 0.f;
        for (int k = lane; k < pe.y; k += 32) {
            const float a = A.rval[pe.x + k];
            acc = fmaf(a * a, A.lam[A.ridx[pe.x + k]], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) A.th[s] = acc;
    }
}

// Super-voxel batch constants from the lane-per-view layout: theta2_p = sum a_p^2 lambda
// (icd.py:193-195) for the kSvBatch slots of each batch, and the cross terms
// c_ij = sum_r a_ir a_jr lambda_r that couple two pixels of a batch through shared rows (k_sv.cuh).
// Depends on lambda only, so it is recomputed per data load.
//
// One 128-thread block per (agent, tile) item.  The tile's lambda band window (the rows its views
// touch, [g][o][32] as in K2's shared-memory plane) is staged once in shared memory, so the
// per-record lambda reads are bank-conflict-free shared loads instead of one scattered L2 sector
// per (lane, record); each warp then streams the slot records of every 4th batch, the next
// batch's records in flight while the current one is reduced.  Weighted contexts (kW) write the
// records back as a sqrt(lambda); plain ones copy the window out as the lambda band K2 stages.
template <int K, int NG>
__device__ __forceinline__ void sv_load_recs(const uint32_t* __restrict__ rb, int lane, float (&a)[4][NG][K],
                                             uint32_t (&ow)[4])
{
    // one (batch, chunk) block, lane-major (internal.h sv_len_word / sv_ofs_word): per group the
    // lane's 4 K lengths are contiguous, its four offset words too (streaming loads)
#if !MACE_SV_LANE_MAJOR
    constexpr int recw = NG * 32 * K + 32;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const uint32_t* r = rb + (size_t)p * recw;
        ow[p] = __ldcs(r + NG * 32 * K + lane);
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int q = 0; q < K; ++q) a[p][g][q] = __uint_as_float(__ldcs(r + (g * 32 + lane) * K + q));
    }
    return;
#endif
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        const uint4* q = reinterpret_cast<const uint4*>(rb + ((size_t)g * 32 + lane) * 4 * K);
#pragma unroll
        for (int h = 0; h < K; ++h) {  // 4 words per load: elements 4h .. 4h + 3 of [slot][k]
            const uint4 v = __ldcs(q + h);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) a[(4 * h + i) / K][g][(4 * h + i) % K] = __uint_as_float(w[i]);
        }
    }
    const uint4 o = __ldcs(reinterpret_cast<const uint4*>(rb + (size_t)NG * 32 * 4 * K) + lane);
    ow[0] = o.x;
    ow[1] = o.y;
    ow[2] = o.z;
    ow[3] = o.w;
}

#ifndef MACE_CONSTS_MINB
#define MACE_CONSTS_MINB 4  // resident blocks per SM the register budget (K = 2) is sized for
#endif
template <int K, int NG, bool kW>
__global__ void __launch_bounds__(128, K == 2 ? MACE_CONSTS_MINB : 1) k_sv_consts(const AgentDev* agents, int n_items, const uint32_t* queue,
                                                   int n_side, int S, int nb, int W, int CH)
{
    extern __shared__ float s_lam[];  // [CH * NG][W][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x;
    if (item >= n_items) return;
    const int h = S / 2, per_class = h * h, bpc = (per_class + 3) / 4;
    constexpr int recw = NG * 32 * K + 32;
    const uint32_t code = queue[item];
    const AgentDev& A = agents[code >> kAgentShift];
    const int sv = (int)(code & kSvMask);
    const int r0 = (sv / A.n_sv_side) * S, c0 = (sv % A.n_sv_side) * S;
    // records: (batch, chunk) blocks of 4 recw words (internal.h); this warp takes batches b = warp + 4 k, and for each
    // the CH chunks (units u = k CH + c), the next unit's records in flight
    const uint32_t* __restrict__ rbase = A.rec0 + (size_t)sv * nb * CH * 4 * recw;
    uint32_t* __restrict__ wbase = kW ? A.recw + (size_t)sv * nb * CH * 4 * recw : nullptr;
    auto unit_ofs = [&](int u) { return ((size_t)(warp + 4 * (u / CH)) * CH + u % CH) * 4 * recw; };  // (batch, chunk) block
    const int nu = (warp < nb ? (nb - warp + 3) / 4 : 0) * CH;

    // first unit's records in flight while the window is staged
    float a[4][NG][K];
    uint32_t ow[4];
    if (nu > 0) sv_load_recs<K, NG>(rbase + unit_ofs(0), lane, a, ow);

    const int2* bt = A.band + (size_t)sv * A.V;
    for (int g = warp; g < CH * NG; g += 4) {
        const int j = 32 * g + lane;
        const int2 bj = j < A.V ? bt[j] : make_int2(0, 0);
        float* sl = s_lam + (size_t)g * W * 32 + lane;
#pragma unroll 8
        // weighted records: the window holds sqrt(lambda) (k_gather_data's A.sq), so a record is
        // weighted by one multiply instead of an IEEE sqrtf per entry
        const float* src = kW ? A.sq : A.lam;
        for (int o = 0; o < W; ++o) sl[o * 32] = o < bj.y ? src[bj.x + o] : 0.f;
    }
    __syncthreads();
    if (!kW) {  // the band's lambda rows, laid out as the K2 shared-memory plane
        float* lb = A.lb + (size_t)sv * CH * NG * W * 32;
        for (int i = threadIdx.x; i < CH * NG * W * 32; i += blockDim.x) lb[i] = s_lam[i];
    }

    float t2[4] = {0.f, 0.f, 0.f, 0.f}, cx[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int u = 0; u < nu; ++u) {
        const int b = warp + 4 * (u / CH), ch = u % CH;
        float an[4][NG][K];
        uint32_t own[4];
        if (u + 1 < nu) sv_load_recs<K, NG>(rbase + unit_ofs(u + 1), lane, an, own);
        float l[4][NG][K];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const float* sl = s_lam + ((size_t)(ch * NG + g) * W + ((ow[p] >> (8 * g)) & 0xffu)) * 32 + lane;
#pragma unroll
                for (int q = 0; q < K; ++q) l[p][g][q] = a[p][g][q] != 0.f ? sl[q * 32] : 0.f;
            }
        if (kW) {  // weighted record a sqrt(lambda): theta2 and the cross terms are its plain products
            uint32_t* wb = wbase + unit_ofs(u);
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) {
                        a[p][g][q] *= l[p][g][q];  // l = sqrt(lambda) here
                        l[p][g][q] = 1.f;
                    }
#if !MACE_SV_LANE_MAJOR
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                uint32_t* w = wb + (size_t)p * recw;
                __stcs(w + NG * 32 * K + lane, ow[p]);
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q = 0; q < K; ++q) __stcs(w + (g * 32 + lane) * K + q, __float_as_uint(a[p][g][q]));
            }
            if (false)
#endif
#pragma unroll
            for (int g = 0; g < NG; ++g) {  // the same lane-major block: 4 K words per (group, lane)
                uint4* q = reinterpret_cast<uint4*>(wb + ((size_t)g * 32 + lane) * 4 * K);
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    uint32_t w[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) w[i] = __float_as_uint(a[(4 * h + i) / K][g][(4 * h + i) % K]);
                    __stcs(q + h, make_uint4(w[0], w[1], w[2], w[3]));
                }
            }
            if (MACE_SV_LANE_MAJOR)
                __stcs(reinterpret_cast<uint4*>(wb + (size_t)NG * 32 * 4 * K) + lane,
                       make_uint4(ow[0], ow[1], ow[2], ow[3]));
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            int o[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                o[p] = (int)((ow[p] >> (8 * g)) & 0xffu);
#pragma unroll
                for (int q = 0; q < K; ++q) t2[p] = fmaf(a[p][g][q] * a[p][g][q], l[p][g][q], t2[p]);
            }
            int x = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = i + 1; j < 4; ++j, ++x) {
                    if constexpr (K == 2) {  // rows shared when |o_j - o_i| <= 1: selects, no branches
                        const int d = o[j] - o[i];
                        const float s0 = a[i][g][0] * l[i][g][0], s1 = a[i][g][1] * l[i][g][1];
                        const float t = d == 0 ? fmaf(s0, a[j][g][0], s1 * a[j][g][1])
                                               : d == 1 ? s1 * a[j][g][0] : d == -1 ? s0 * a[j][g][1] : 0.f;
                        cx[x] += t;
                    } else {
#pragma unroll
                        for (int q = 0; q < K; ++q)
#pragma unroll
                            for (int qj = 0; qj < K; ++qj)  // row o_i + q of pixel i is row o_j + qj of pixel j
                                if (o[i] + q == o[j] + qj) cx[x] = fmaf(a[i][g][q] * a[j][g][qj], l[i][g][q], cx[x]);
                    }
                }
        }
        if (ch == CH - 1) {  // the batch's sums over every chunk's views
            // the ten sums at once by a halving butterfly: at the xor-m stage a lane keeps the half of
            // its values selected by its lane bit m and adds the partner's copy of that half; after
            // the xor-2 stage value k sits on lanes 2k and 2k + 1 (16 shuffles instead of 50)
            float r16[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) r16[k] = k < 4 ? t2[k] : (k < 10 ? cx[k - 4] : 0.f);
#pragma unroll
            for (int m = 16, h = 8; m >= 2; m >>= 1, h >>= 1) {
                const bool up = lane & m;
#pragma unroll
                for (int k = 0; k < h; ++k) {
                    const float send = up ? r16[k] : r16[k + h];
                    const float keep = up ? r16[k + h] : r16[k];
                    r16[k] = keep + __shfl_xor_sync(FULL, send, m);
                }
            }
            float v = r16[0] + __shfl_xor_sync(FULL, r16[0], 1);  // value lane >> 1
            v = __shfl_sync(FULL, v, 2 * (lane & 15));             // lane k (< 16) takes value k
            if (lane < 16) A.bc[((size_t)sv * nb + b) * 16 + lane] = lane < 10 ? v : 0.f;
            if (lane < 4) {  // theta2 image (cost kernels, diagnostics)
                const int i = (b % bpc) * 4 + lane, cls = b / bpc;
                if (i < per_class) {
                    const int lr = (cls >> 1) + 2 * (i / h), lc = (cls & 1) + 2 * (i % h);
                    if (r0 + lr < n_side && c0 + lc < n_side) A.th[(size_t)(r0 + lr) * n_side + c0 + lc] = v;
                }
            }
#pragma unroll
            for (int p = 0; p < 4; ++p) t2[p] = 0.f;
#pragma unroll
            for (int x = 0; x < 6; ++x) cx[x] = 0.f;
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            ow[p] = own[p];
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int q = 0; q < K; ++q) a[p][g][q] = an[p][g][q];
        }
    }
}

// agent rows <- global y / lambda (local row r = j n_ch + c, icd.py:187-188)
__global__ void k_gather_data(const AgentDev* agents, const int* row_base, int n_agents, int total_rows, int n_ch,
                              const float* y, const float* lam, int64_t slice_rows)
{
    for (int wr = blockIdx.x * blockDim.x + threadIdx.x; wr < total_rows; wr += gridDim.x * blockDim.x) {
        const int a = agent_of_row(row_base, n_agents, wr);
        const AgentDev& A = agents[a];
        const int r = wr - row_base[a];
        if (r >= A.R) continue;
        const int64_t g = (int64_t)A.slice * slice_rows + (int64_t)A.views[r / n_ch] * n_ch + r % n_ch;
        A.y[r] = y[g];
        A.lam[r] = lam[g];
        if (A.sq) A.sq[r] = sqrtf(lam[g]);
    }
}

// ===========================================================================
// K4: consensus average in the reference's fixed pairwise-tree order
// (mace.py:71-90), optionally the local partial sum for multi-rank runs.
// W is [group][n_local][n] (a group = one slice of a multi-slice batch); out is [group][n].
// ===========================================================================
// Fixed-order pairwise tree over m agent values (mace.py:71-90): halve, folding the odd tail.
// With M a compile-time count every index is static and the values stay in registers.
template <int M>
__device__ __forceinline__ float tree_sum(float* acc)
{
    int m = M;
#pragma unroll
    for (int r = 0; r < 12; ++r) {
        if (m <= 1) break;
        const int half = m / 2;
#pragma unroll
        for (int i = 0; i < half; ++i) acc[i] += acc[half + i];
        if (m % 2) {
            acc[half] = acc[2 * half];
            m = half + 1;
        } else {
            m = half;
        }
    }
    return acc[0];
}

// NL > 0: exactly NL agents (register tree); NL == 0: any n_local <= 64 (local-memory tree)
template <int NL>
__global__ void k_consensus(const float* W, int n_local, size_t n, float scale, float* out, const float* ref,
                            double* ref_part, const int* done, int n_groups)
{
    if (done && *done) return;
    double loc = 0.0;
    for (size_t gs = blockIdx.x * (size_t)blockDim.x + threadIdx.x; gs < n * n_groups;
         gs += (size_t)gridDim.x * blockDim.x) {
        const size_t grp = gs / n, s = gs % n;
        const float* Wg = W + grp * n_local * n;
        float v;
        if constexpr (NL > 0) {
            float acc[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) acc[i] = __ldcg(Wg + (size_t)i * n + s);
            v = tree_sum<NL>(acc) / scale;
        } else {
            float acc[64];
            for (int i = 0; i < n_local; ++i) acc[i] = Wg[(size_t)i * n + s];
            int m = n_local;
            while (m > 1) {
                const int half = m / 2;
                for (int i = 0; i < half; ++i) acc[i] += acc[half + i];
                if (m % 2) {
                    acc[half] = acc[2 * half];
                    m = half + 1;
                } else {
                    m = half;
                }
            }
            v = acc[0] / scale;
        }
        out[gs] = v;
        if (ref && grp == 0) {
            const double d = (double)v - (double)ref[s];
            loc += d * d;
        }
    }
    if (ref_part) {
        __shared__ double sh[256];
        sh[threadIdx.x] = loc;
        __syncthreads();
        for (int o = blockDim.x / 2; o; o >>= 1) {
            if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) ref_part[blockIdx.x] = sh[0];
    }
}

// Fixed-order reduction of the per-item partials -> out5[0..3] (and the nrmse^2 partials
// -> out5[4]).  Each block folds a contiguous slice into scratch[5 * block]; the last
// block to finish folds the block sums in block order, so the result is deterministic.
__global__ void k_norms(const double* part, int n_items, const double* ref_part, int n_ref, double* scratch,
                        double* out5, unsigned* counter, const int* done)
{
    if (done && *done) return;
    __shared__ double sh[5][256];
    __shared__ bool last;
    double a[5] = {0, 0, 0, 0, 0};
    const int chunk = (n_items + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * chunk, i1 = min(n_items, i0 + chunk);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        for (int k = 0; k < 4; ++k) a[k] += part[(size_t)i * 4 + k];
    if (ref_part && blockIdx.x == 0)
        for (int i = threadIdx.x; i < n_ref; i += blockDim.x) a[4] += ref_part[i];
    for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o)
            for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < 5; ++k) scratch[5 * blockIdx.x + k] = sh[k][0];
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {  // fixed-order tree over the block sums (gridDim.x <= blockDim.x)
        for (int k = 0; k < 5; ++k)
            sh[k][threadIdx.x] = (int)threadIdx.x < (int)gridDim.x ? __ldcg(scratch + 5 * threadIdx.x + k) : 0.0;
        __syncthreads();
        for (int o = blockDim.x / 2; o; o >>= 1) {
            if ((int)threadIdx.x < o)
                for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            for (int k = 0; k < 5; ++k) out5[k] = sh[k][0];
            *counter = 0u;
        }
    }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// relnorm, divergence and stop test (mace.py:309-318,337-339); log row [relnorm, |w'|, sum a^2, nrmse^2]
// ctr != nullptr: the iteration index comes from (and advances) a device counter, so a CUDA graph of
// several iterations needs no per-iteration host argument
__global__ void k_finish(const double* sums5, double ref_norm2, double tol, int iter, double* log, int* done,
                         unsigned* head, int* ctr = nullptr)
{
    if (*done) return;
    if (ctr) iter = (*ctr)++;
    const double dw2 = sums5[1], wn2 = sums5[2], wo2 = sums5[3];
    const double nn = sqrt(wn2);
    const double rel = sqrt(dw2) / fmax(sqrt(wo2), 1e-300);
    double* L = log + (size_t)iter * 4;
    L[0] = rel;
    L[1] = nn;
    L[2] = sums5[0];
    L[3] = ref_norm2 > 0.0 ? sqrt(sums5[4] / ref_norm2) : -1.0;
    if (!isfinite(nn)) {
        done[0] = 2;
        done[1] = iter + 1;
    } else if (rel < tol) {
        done[0] = 1;
        done[1] = iter + 1;
    }
    *head = 0u;
}

// The tail of one single-context MACE iteration in one launch: the consensus average (K4 tree,
// optionally the NRMSE partials against ref), the per-item norm partials of K2 folded per block, and
// in the last block to finish a fixed-order fold of the block sums followed by the stop test and log
// row (k_finish).  Same arithmetic order as k_consensus + k_norms + k_finish; gridDim <= 256.
template <int NL>
__global__ void __launch_bounds__(256) k_tail(const float* __restrict__ W, int n_local, size_t n, float scale,
                                              float* __restrict__ out, const float* __restrict__ ref,
                                              const double* __restrict__ part, int n_items, double* scratch,
                                              unsigned* counter, double* sums5, double ref_norm2, double tol,
                                              int iter, double* log, int* done, unsigned* head, int n_groups)
{
    if (*done) return;
    __shared__ double sh[5][256];
    __shared__ bool last;
    double a[5] = {0, 0, 0, 0, 0};
    // NL > 0 and n a multiple of 4: four pixels per thread, 128-bit loads and stores (the same tree per pixel)
    const bool vec4 = NL > 0 && (n & 3) == 0;
    if constexpr (NL > 0) {
        if (vec4) {
            const size_t nq = n / 4;
            for (size_t gq = blockIdx.x * (size_t)blockDim.x + threadIdx.x; gq < nq * n_groups;
                 gq += (size_t)gridDim.x * blockDim.x) {
                const size_t grp = gq / nq, s = (gq % nq) * 4;
                const float* Wg = W + grp * n_local * n;
                float4 q[NL];
#pragma unroll
                for (int i = 0; i < NL; ++i) q[i] = __ldcg(reinterpret_cast<const float4*>(Wg + (size_t)i * n + s));
                float acc[NL];
                float4 v;
#pragma unroll
                for (int i = 0; i < NL; ++i) acc[i] = q[i].x;
                v.x = tree_sum<NL>(acc) / scale;
#pragma unroll
                for (int i = 0; i < NL; ++i) acc[i] = q[i].y;
                v.y = tree_sum<NL>(acc) / scale;
#pragma unroll
                for (int i = 0; i < NL; ++i) acc[i] = q[i].z;
                v.z = tree_sum<NL>(acc) / scale;
#pragma unroll
                for (int i = 0; i < NL; ++i) acc[i] = q[i].w;
                v.w = tree_sum<NL>(acc) / scale;
                *reinterpret_cast<float4*>(out + grp * n + s) = v;
                if (ref && grp == 0) {
                    const float4 r4 = *reinterpret_cast<const float4*>(ref + s);
                    const double d0 = (double)v.x - (double)r4.x, d1 = (double)v.y - (double)r4.y;
                    const double d2 = (double)v.z - (double)r4.z, d3 = (double)v.w - (double)r4.w;
                    a[4] += d0 * d0;
                    a[4] += d1 * d1;
                    a[4] += d2 * d2;
                    a[4] += d3 * d3;
                }
            }
        }
    }
    for (size_t gs = blockIdx.x * (size_t)blockDim.x + threadIdx.x; !vec4 && gs < n * n_groups;
         gs += (size_t)gridDim.x * blockDim.x) {
        const size_t grp = gs / n, s = gs % n;
        const float* Wg = W + grp * n_local * n;
        float v;
        if constexpr (NL > 0) {
            float acc[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) acc[i] = __ldcg(Wg + (size_t)i * n + s);
            v = tree_sum<NL>(acc) / scale;
        } else {
            float acc[64];
            for (int i = 0; i < n_local; ++i) acc[i] = Wg[(size_t)i * n + s];
            int m = n_local;
            while (m > 1) {
                const int half = m / 2;
                for (int i = 0; i < half; ++i) acc[i] += acc[half + i];
                if (m % 2) {
                    acc[half] = acc[2 * half];
                    m = half + 1;
                } else {
                    m = half;
                }
            }
            v = acc[0] / scale;
        }
        out[gs] = v;
        if (ref && grp == 0) {
            const double d = (double)v - (double)ref[s];
            a[4] += d * d;
        }
    }
    const int chunk = (n_items + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * chunk, i1 = min(n_items, i0 + chunk);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        for (int k = 0; k < 4; ++k) a[k] += part[(size_t)i * 4 + k];
    for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o)
            for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < 5; ++k) scratch[5 * blockIdx.x + k] = sh[k][0];
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    for (int k = 0; k < 5; ++k) {  // the block sums, gridDim <= 1024: a fixed-order fold in 256 lanes
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += __ldcg(scratch + 5 * b + k);
        sh[k][threadIdx.x] = v;
    }
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o)
            for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < 5; ++k) sums5[k] = sh[k][0];
        *counter = 0u;
        const double dw2 = sh[1][0], wn2 = sh[2][0], wo2 = sh[3][0];
        const double nn = sqrt(wn2);
        const double rel = sqrt(dw2) / fmax(sqrt(wo2), 1e-300);
        double* L = log + (size_t)iter * 4;
        L[0] = rel;
        L[1] = nn;
        L[2] = sh[0][0];
        L[3] = ref_norm2 > 0.0 ? sqrt(sh[4][0] / ref_norm2) : -1.0;
        if (!isfinite(nn)) {
            done[0] = 2;
            done[1] = iter + 1;
        } else if (rel < tol) {
            done[0] = 1;
            done[1] = iter + 1;
        }
        *head = 0u;
    }
}

__global__ void k_reset_head(unsigned* head) { *head = 0u; }

// deterministic mode, after each colour class: e += fixed-point deltas (then zeroed)
__global__ void k_fold_delta(float* __restrict__ e, unsigned long long* __restrict__ ed, int rows, const int* done)
{
    if (done && *done) return;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const unsigned long long q = ed[r];
        if (q) {
            e[r] += (float)((double)(long long)q * (1.0 / kDetScale));
            ed[r] = 0ull;
        }
    }
}

__global__ void k_fill(float* p, size_t n, float v)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// out = a * b elementwise (weighted error sinogram of a zero state: sqrt(lambda) y)
__global__ void k_mul(float* out, const float* a, const float* b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = a[i] * b[i];
}

// X_i = x[slice(i)] for every local (virtual) agent; x is [slice][n]
__global__ void k_broadcast_state(const AgentDev* agents, int n_agents, const float* x, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n * n_agents; i += (size_t)gridDim.x * blockDim.x) {
        const AgentDev& A = agents[i / n];
        A.z[i % n] = x[(size_t)A.slice * n + i % n];
    }
}

}  // namespace mace
