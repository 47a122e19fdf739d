// Device types and inline helpers shared by every translation unit of libmace_b200
// (mace.cu and the per-tile-side K2 units k2_inst.cu): agent/pass parameter blocks,
// prior constants (models.py:50-52), the qGGMRF derivatives (icd.py:45-64) and warp sums.
// Everything here is inline or TU-local (static __constant__), so each unit carries its own copy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// slot-record block layout (internal.h sv_len_word): 1 = lane-major (default), 0 = slot-major
#ifndef MACE_SV_LANE_MAJOR
#define MACE_SV_LANE_MAJOR 1
#endif

namespace mace {

constexpr unsigned FULL = 0xffffffffu;
// work-queue item = (local agent << kAgentShift) | super-voxel index (layout.cpp build_queue)
constexpr int kAgentShift = 22;
constexpr uint32_t kSvMask = (1u << kAgentShift) - 1;

struct PriorC {
    int kind;  // 0 quadratic-mrf, 1 qggmrf  (models.py:43-44)
    int p_is_2;
    float eps2;      // 2 * eps_reg
    float inv_Tsx;   // 1 / (T sigma_x)
    float inv_sxp;   // sigma_x^-p
    float qp;        // q / p
    float qmp;       // q - p
    float pm1, pm2;  // p - 1, p - 2
    float floor_;    // 1e-9 T sigma_x
    float inv_sx2;   // 1 / sigma_x^2
    double p, q, T, sx, eps;  // double copies for the cost kernels
};

struct AgentDev {
    float* e;          // [R] error sinogram y_i - A_i X_i (icd.py:200); sqrt(lambda) (y_i - A_i X_i) if sq
    float* lam;        // [R] weights lambda
    float* sq;         // [R] sqrt(lambda) when K2 runs weighted records (k_sv.cuh), else nullptr
    float* y;          // [R]
    float* z;          // [n] agent state X_i
    float* w;          // [n] stack component w_i
    float* th;         // [n] theta2 data term, sum a^2 lambda (icd.py:193-195)
    float* vt;         // [n] explicit proximal target (plain passes)
    int slice;         // slice of a multi-slice batch (config 4); consensus images are [slice][n]
    const int* views;  // [V] global view index of local view j
    // super-voxel layout
    const int2* band;      // [n_sv * V] {local row start, window rows}
    const uint32_t* rec;   // [n_sv][nb][4][rec_words] slot records K2 reads (lengths a, or a sqrt(lambda))
    const uint32_t* rec0;  // the plain records (layout.cpp, lane-per-view)
    uint32_t* recw;        // weighted records k_sv_consts writes (== rec when sq != nullptr, else nullptr)
    float* bc;             // [n_sv][nb][16] batch constants: theta2 x4, cross terms x6 (per local agent)
    unsigned long long* ed;  // [R] deterministic mode: fixed-point e deltas of the running colour class
    float* lb;             // [n_sv][ng][wcap][32] band lambda in shared-memory order (per local agent)
    int ng, rec_words;     // view groups ceil(V / 32); words per slot record
    // raster layout
    const int2* rpix;   // [n]
    const uint32_t* ridx;
    const float* rval;
    int R, V, n_sv_side;
    float beta_eff, inv_s2;
    int clamp;
};

struct PassParams {
    const AgentDev* agents;
    PriorC pr;
    int n_side, S, mode;  // mode 0: v from vt; 1: MACE (v = 2 g - w, Mann epilogue)
    const float* g;       // consensus image G(w) or G_H(w)
    float rho;
    const uint32_t* queue;
    int n_items;
    unsigned* head;
    double* part;  // [n_items * 4]: sum alpha^2, sum (w'-w)^2, sum w'^2, sum w^2
    int ng, wcap;  // shared-memory band geometry (max over agents)
    int chunks;    // view chunks (warps) per super-voxel tile: 1, or > 1 for agents with > 128 views
    int det;       // deterministic class-synchronous mode: write-back into AgentDev::ed (fixed point)
    const int* done;
    long s_begin, s_end;  // raster passes: pixel range [s_begin, s_end) (icd.py:222-246)
};

// deterministic mode: e deltas accumulated as signed 2^-40 fixed point (k_sv.cuh write-back,
// k_fold_delta); |delta| < 2^23 per row and class, resolution 9e-13
constexpr double kDetScale = 1099511627776.0;

static __constant__ int c_dr[8] = {-1, -1, -1, 0, 0, 1, 1, 1};  // models.py:50
static __constant__ int c_dc[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
// raw weight (1 or 1/sqrt 2) / (4 + 2 sqrt 2), models.py:51-52,107, rounded once from double
// (the same floats as (float)(raw / norm) with std::sqrt on the host)
constexpr double kInvSqrt2 = 0.70710678118654752440, kNbrNorm = 6.82842712474619009760;
static __constant__ float c_nw[8] = {(float)(kInvSqrt2 / kNbrNorm), (float)(1.0 / kNbrNorm), (float)(kInvSqrt2 / kNbrNorm),
                                     (float)(1.0 / kNbrNorm),       (float)(1.0 / kNbrNorm), (float)(kInvSqrt2 / kNbrNorm),
                                     (float)(1.0 / kNbrNorm),       (float)(kInvSqrt2 / kNbrNorm)};

// ---- qGGMRF potential derivatives in fp32 (icd.py:45-64)
__device__ __forceinline__ float pow_pos(float x, float e) { return exp2f(e * log2f(x)); }

__device__ __forceinline__ float qg_influence(float d, const PriorC& P)
{
    const float ad = fabsf(d);
    if (ad == 0.0f) return 0.0f;
    const float um = pow_pos(ad * P.inv_Tsx, P.qmp);
    const float base = P.p_is_2 ? ad : pow_pos(ad, P.pm1);
    const float opu = 1.0f + um;
    const float val = (base * P.inv_sxp) * um * (P.qp + um) / (opu * opu);
    return d > 0.0f ? val : -val;
}

__device__ __forceinline__ float qg_coef(float d, const PriorC& P)
{
    float ad = fabsf(d);
    if (ad <= P.floor_) {
        if (P.p_is_2) return P.inv_sx2;
        ad = P.floor_;
    }
    const float um = pow_pos(ad * P.inv_Tsx, P.qmp);
    const float base = P.p_is_2 ? 1.0f : pow_pos(ad, P.pm2);
    const float opu = 1.0f + um;
    return (base * P.inv_sxp) * um * (P.qp + um) / (opu * opu);
}

__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Neighbour term of one lane (lanes 0..7 own neighbour k = lane; models.py:50-52 order).
__device__ __forceinline__ void prior_lane(int lane, float zs, float zr, bool valid, const PriorC& P,
                                           float& g, float& c)
{
    g = 0.f;
    c = 0.f;
    if (lane < 8 && valid) {
        const float wk = c_nw[lane];
        if (P.kind == 0) {
            g = wk * (zs - zr);
            c = wk;
        } else {
            const float d = zs - zr;
            g = wk * qg_influence(d, P);
            c = wk * qg_coef(d, P);
        }
    }
}

// 1-D surrogate solve (icd.py:128-134); returns false where the reference `continue`s.
__device__ __forceinline__ bool pixel_step(float t, float g, float c, float zs, float v, float th, float beta,
                                           float inv_s2, int clamp, const PriorC& P, float& alpha)
{
    float gp = 0.f, cp = 0.f;
    if (beta > 0.f) {
        if (P.kind == 0) {
            gp = beta * (g + P.eps2 * zs);
            cp = beta * (c + P.eps2);
        } else {
            gp = beta * g;
            cp = beta * c;
        }
    }
    const float num = t - gp - inv_s2 * (zs - v);
    const float den = th + cp + inv_s2;
    if (!(den > 0.f)) return false;
    alpha = num / den;
    if (clamp && zs + alpha < 0.f) alpha = -zs;
    return true;
}

}  // namespace mace
