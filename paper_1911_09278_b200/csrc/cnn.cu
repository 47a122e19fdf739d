// K5: the PnP denoiser H of MACE-PnP (mace.py:105-108, applied to the consensus average)
// as a 17-layer bias-free 3x3 conv net, 64 channels, ReLU, out = x - net(x), bf16 weights
// and bf16 activations between layers, fp32 accumulation (BASELINE config 3).
//
// Layers 2..16 (64 -> 64) run on the 5th-gen tensor cores: an implicit GEMM per output row
// segment of 128 pixels, D[128 px x 64 oc] = sum over 9 taps and 4 K-steps of
// A[128 px x 16 ic] * W[16 ic x 64 oc]  (tcgen05.mma.cta_group::1.kind::f16, M=128, N=64,
// K=16, fp32 accumulators in TMEM).  Activations live in HBM channel-blocked,
// [8 channel groups][H][W][8 ch] bf16, so a halo row ([8 groups][130 px][8 ch], 16.6 KB) is
// 8 contiguous 2 KB runs: one 4-D TMA box (out-of-image coordinates are zero-filled = the
// conv's zero padding).  The tap shift dx is a 16-byte offset of the UMMA descriptor
// (SWIZZLE_NONE, K-major, core matrix = 8 px x 8 ch).  The 9 taps' weights (72 KB) stay
// resident in shared memory.  A warp-specialized pipeline (TMA producer, MMA issuer, 4
// epilogue warps: tcgen05.ld -> ReLU -> bf16 -> blocked stores) keeps 4 accumulators in flight.
// Layers 1 (1 -> 64) and 17 (64 -> 1, fused residual) are CUDA-core kernels.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "cnn.cuh"

namespace mace {

namespace {

constexpr int kC = 64;             // channels
constexpr int kTileX = 128;        // output pixels per tile (one row segment)
// halo row in shared memory: 18 chunks of 8 px from x0 - 8 (TMA moves whole 128-byte chunks;
// the 3x3 window spans pixels x0 - 1 .. x0 + 128, i.e. slot pixels 7 .. 136)
constexpr int kHaloX = kTileX + 16;  // 144
constexpr int kHaloOff = 7;         // pixel of the slot that holds x0 - 1
constexpr int kSlots = 8;          // ring of halo rows (row pairs consume two per unit: 8 keeps TMA a unit ahead)
constexpr int kAcc = 4;            // TMEM accumulators (4 x 64 fp32 columns)
constexpr int kSlotBytes = 8 * kHaloX * 16;         // 18,432
constexpr int kWBytes = 9 * kC * kC * 2;            // 73,728
constexpr int kSmem = kWBytes + kSlots * kSlotBytes + 1024;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(s_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_row(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar)
{
    // 4-D box {64 = 8 px x 8 ch, 18 chunks, 1 row, 8 groups} at (0, x chunk, y, 0)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(s_u32(dst)),
        "l"(map), "r"(0), "r"(x), "r"(y), "r"(0), "r"(s_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s_u32(dst)),
                 "l"(src), "r"(bytes), "r"(s_u32(bar))
                 : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major (cute/arch/mma_sm100_desc.hpp layout):
// start>>4 [0,14), LBO>>4 [16,30) (K-adjacent core matrices), SBO>>4 [32,46) (8-row groups),
// version 1 at [46,48), layout type 0 at [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

// instruction descriptor: D f32, A/B bf16, both K-major, N = 64, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

// Warp-wide forms: the whole issuer warp runs the loop (so descriptor arithmetic stays in uniform
// registers) and one elected lane issues; issuing from a single divergent lane made every
// descriptor cross from the vector to the uniform register file (R2UR) in front of each UMMA.
__device__ __forceinline__ void umma_e(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate)
{
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_e(uint64_t* bar)
{
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(s_u32(bar))
        : "memory");
}

#define LD16(base, r)                                                                                             \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
                 "[%16];"                                                                                         \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
                   "=r"(r[14]), "=r"(r[15])                                                                       \
                 : "r"(base))

// One 64->64 conv layer (+ ReLU) over a channel-blocked [8][H][W][8] bf16 image, warp-specialized:
//   warp 0 (one lane)  TMA producer: halo rows y0-1 .. y1 into a ring of kSlots slots
//   warp 1 (one lane)  MMA issuer:   tile y = 36 UMMAs (9 taps x 4 K-steps) into TMEM
//                                    accumulator t % kAcc, commits to acc_full / slot_empty
//   warps 2..5         epilogue:     tcgen05.ld -> ReLU -> bf16 -> blocked stores, acc_empty
// (warp i may only touch TMEM lanes 32*(i%4)..+31, so warps 2..5 cover all 128 rows.)
// Grid: one CTA per (128-px strip, run of rows), one CTA per SM.
#ifdef K5_TRACE  // profiling builds only (tools/micro/k5_trace.cu): per-CTA clock64 timeline of a layer
__device__ long long g_k5_trace[148][64];  // [0] start, [1] weights landed, [2+2t] tile t issued, [3+2t] tile t stored
#define K5T(i) g_k5_trace[blockIdx.x][(i)] = clock64()
#define K5V(i, v) g_k5_trace[blockIdx.x][(i)] = (v)
#define K5ACC(var, stmt)            \
    {                               \
        const long long c_ = clock64(); \
        stmt;                       \
        var += clock64() - c_;      \
    }
__device__ long long g_k5_life[4096][4];  // {smid, start, gdc wait passed, end} in globaltimer ns, one record per CTA
__device__ unsigned g_k5_life_n;
__device__ __forceinline__ long long k5_gtime()
{
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#else
#define K5T(i)
#define K5V(i, v)
#define K5ACC(var, stmt) stmt;
#endif
__global__ void __launch_bounds__(192, 1) k_conv64_tc(const __grid_constant__ CUtensorMap amap,
                                                      const __nv_bfloat16* __restrict__ wts, __nv_bfloat16* out,
                                                      int H, int W, int Wp, int rows_per_cta)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;                     // weights: [tap 9][ic-group 8][oc 64][8 ic]
    unsigned char* slots = sm + kWBytes;        // [slot][ic-group 8][130 px][8 ch]
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;                      // weights landed
    uint64_t* sfull = bars + 1;                 // [kSlots] halo row landed
    uint64_t* sempty = sfull + kSlots;          // [kSlots] halo row no longer read
    uint64_t* afull = sempty + kSlots;          // [kAcc] accumulator ready
    uint64_t* aempty = afull + kAcc;            // [kAcc] accumulator drained (4 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kAcc);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) K5T(0);
    // programmatic dependent launch: the next layer may start its prologue (TMEM, barriers,
    // weights) as soon as SMs free up; it waits for this grid before touching activations
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips;
    const int x0 = strip * kTileX;
    const int y0 = (blockIdx.x / strips) * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    if (y0 >= H) return;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kAcc * 64)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(sempty + i, 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            mbar_init(afull + i, 1);
            mbar_init(aempty + i, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;  // row r -> ring index q = r - rbase, slot q % kSlots, use q / kSlots

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            mbar_expect(wbar, kWBytes);
            bulk_copy(sw, wts, kWBytes, wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous layer's activations
            for (int r = y0 - 1; r <= y1; ++r) {
                const int q = r - rbase, s = q % kSlots, u = q / kSlots;
                if (u >= 1) mbar_wait(sempty + s, (uint32_t)((u - 1) & 1));
                mbar_expect(sfull + s, kSlotBytes);
                if (q < 16) K5T(32 + q);  // TMA issue time of ring row q
                tma_row(slots + s * kSlotBytes, &amap, x0 / 8 - 1, r, sfull + s);
            }
        }
    } else if (warp == 1) {
        {  // ---- MMA issuer (whole warp, one elected lane issues)
            const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
            mbar_wait(wbar, 0);
            if (lane == 0) K5T(1);
            for (int y = y0; y < y1; ++y) {
                const int t = y - y0, b = t % kAcc, ub = t / kAcc;
                if (ub >= 1) mbar_wait(aempty + b, (uint32_t)((ub - 1) & 1));
                for (int r = y - 1; r <= y + 1; ++r) {
                    const int q = r - rbase;
                    mbar_wait(sfull + q % kSlots, (uint32_t)((q / kSlots) & 1));
                    if (lane == 0 && r == y + 1 && q < 16) K5T(48 + q);  // ring row q landed (as seen by the MMA issuer)
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + (uint32_t)(b * 64);
                // descriptors differ only in the start-address field (bits [0,14), addr >> 4):
                // build one per operand and step it with integer adds
                const uint64_t b0 = sdesc(sw_base, kC * 16, 128);
#pragma unroll
                for (int dy = 0; dy < 3; ++dy) {
                    const uint64_t a0 = sdesc(sl_base + ((y - 1 + dy - rbase) % kSlots) * kSlotBytes, kHaloX * 16, 128);
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint64_t a = a0 + (uint64_t)(((kHaloOff + dx) * 16 + 2 * j * (kHaloX * 16)) >> 4);
                            const uint64_t bd = b0 + (uint64_t)(((dy * 3 + dx) * (kC * kC * 2) + 2 * j * (kC * 16)) >> 4);
                            umma_e(d, a, bd, kIdesc, (dy | dx | j) != 0);
                        }
                    }
                }
                umma_commit_e(afull + b);
                umma_commit_e(sempty + (y - 1 - rbase) % kSlots);  // row y-1: last reader was tile y
                if (lane == 0) K5T(2 + 2 * t);
            }
        }
    } else {  // ---- epilogue warps 2..5
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        for (int y = y0; y < y1; ++y) {
            const int t = y - y0, b = t % kAcc, ub = t / kAcc;
            mbar_wait(afull + b, (uint32_t)(ub & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * 64);
            uint32_t r[64];
            LD16(base + 0, (r + 0));
            LD16(base + 16, (r + 16));
            LD16(base + 32, (r + 32));
            LD16(base + 48, (r + 48));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + b)) : "memory");
            const int px = x0 + quad * 32 + lane;
            if (px < W) {
                // channel-blocked output [group][H][Wp][8]: each store is 512 B contiguous per warp
                uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)y * Wp + px);
                const size_t gstride = (size_t)H * Wp;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t pk[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float lo = fmaxf(__uint_as_float(r[8 * q + 2 * h]), 0.f);
                        const float hi = fmaxf(__uint_as_float(r[8 * q + 2 * h + 1]), 0.f);
                        const __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, hi);
                        pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
                    }
                    dst[q * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
            if (warp == 2 && lane == 0) K5T(3 + 2 * t);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * 64) : "memory");
}

// Row-pair variant of the 64->64 layer.  Output rows come in pairs (y, y+1) and their two
// accumulators sit side by side in TMEM, so a halo row that feeds both rows is one N = 128 UMMA
// against two taps' weights stored next to each other: per (dx, K-step) halo rows y and y+1 each
// give one N = 128 UMMA (B = [W_dy1 | W_dy0] and [W_dy2 | W_dy1]) and rows y-1 and y+2 one N = 64
// UMMA each: 48 UMMAs per pair instead of 72 (an N = 128 UMMA costs 64 cycles against 48 for
// N = 64, tools/micro/umma_rate.cu).  Weights: [dx 3][ic-group 8][dy2 | dy1 | dy0 x 64 oc][8 ic].
// A CTA with an odd row count finishes with one single row (N = 64 only).
constexpr uint32_t kIdesc128 =
    (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr int kW2Dx = 8 * 3 * kC * 16;  // 24,576 B per dx: [icg 8][192 oc][8 ic]
constexpr int kW2Icg = 3 * kC * 16;     // 3,072 B per ic-group


constexpr uint32_t kIdesc192 =
    (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(192 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

// One halo row's 12 UMMAs (3 dx shifts x 4 K-steps) from one elected lane in a single asm block:
// the descriptors step by compile-time offsets (A: dx + 2 j x 144 px rows, B: dx x 24,576 B + 2 j x
// 3,072 B, all >> 4), so only the two base descriptors cross into uniform registers per row.
__device__ __forceinline__ void umma_row12(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t accumulate)
{
    static_assert(kHaloX == 144 && kW2Dx == 24576 && kW2Icg == 3072, "offsets below are hard-coded");
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 1, 1;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "add.s64 a, %1, 288;\nadd.s64 b, %2, 384;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 576;\nadd.s64 b, %2, 768;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 864;\nadd.s64 b, %2, 1152;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 1;\nadd.s64 b, %2, 1536;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 289;\nadd.s64 b, %2, 1920;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 577;\nadd.s64 b, %2, 2304;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 865;\nadd.s64 b, %2, 2688;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 2;\nadd.s64 b, %2, 3072;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 290;\nadd.s64 b, %2, 3456;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 578;\nadd.s64 b, %2, 3840;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 866;\nadd.s64 b, %2, 4224;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate)
        : "memory");
}

// R = 2 (row pairs) or 3 (row triples: the middle halo row feeds all three rows through one
// N = 192 UMMA against [W_dy2 | W_dy1 | W_dy0]; 80 UMMAs per 3 rows)
template <int R>
__global__ void __launch_bounds__(192, 1) k_conv64_tc2(const __grid_constant__ CUtensorMap amap,
                                                       const __nv_bfloat16* __restrict__ wts, __nv_bfloat16* out,
                                                       int H, int W, int Wp, int rows_per_cta)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;
    unsigned char* slots = sm + kWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;
    uint64_t* sfull = bars + 1;
    uint64_t* sempty = sfull + kSlots;
    uint64_t* afull = sempty + kSlots;   // [2] accumulator pair ready
    uint64_t* aempty = afull + kAcc;     // [2] accumulator pair drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kAcc);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        K5T(0);
        K5V(48, k5_gtime());
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips;
    const int x0 = strip * kTileX;
    const int y0 = (blockIdx.x / strips) * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    if (y0 >= H) return;
    const int n_units = (y1 - y0 + R - 1) / R;  // R-row units, the last one possibly shorter
    constexpr int kAccCols = R == 2 ? 256 : 512;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kAccCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(sempty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(afull + i, 1);
            mbar_init(aempty + i, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (as k_conv64_tc)
            mbar_expect(wbar, kWBytes);
            bulk_copy(sw, wts, kWBytes, wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");
            K5T(30);
            for (int r = y0 - 1; r <= y1; ++r) {
                const int q = r - rbase, s = q % kSlots, u = q / kSlots;
#ifdef K5_NO_TMA  // timing experiment only: the ring is filled once, later rows reuse what is there
                if (q >= kSlots) break;
#endif
                if (u >= 1) mbar_wait(sempty + s, (uint32_t)((u - 1) & 1));
                mbar_expect(sfull + s, kSlotBytes);
                tma_row(slots + s * kSlotBytes, &amap, x0 / 8 - 1, r, sfull + s);
            }
        }
    } else if (warp == 1) {
        {  // ---- MMA issuer (whole warp, one elected lane issues)
            const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
            mbar_wait(wbar, 0);
            if (lane == 0) K5T(1);
            int landed = y0 - 2;  // halo rows <= landed are known to be in shared memory
            [[maybe_unused]] long long st_full = 0, st_acc = 0, st_issue = 0;
            for (int t = 0; t < n_units; ++t) {
                const int y = y0 + R * t, b = t & 1, ub = t >> 1;
                const int nr = min(R, y1 - y);  // rows in this unit
                if (ub >= 1) {
                    K5ACC(st_acc, mbar_wait(aempty + b, (uint32_t)((ub - 1) & 1)))
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                const uint32_t d = tmem + (uint32_t)(b * R * 64);
#ifdef K5_TRACE
                int rstamp = 19;
                if (t == 2 && lane == 0) K5T(18);
#endif
                // one halo row r against weight block blk (0 = dy2, 1 = dy1, 2 = dy0) with N = 64 or 128
                auto row = [&](int r, int blk, uint32_t dcol, uint32_t idesc, bool first) {
                    // wait for halo rows just before their first UMMAs, so the UMMAs already queued keep
                    // the tensor pipe busy meanwhile (rows y+1.. of a unit were waited for by the last one)
                    if (r > landed) {
                        while (landed < r) {
                            ++landed;
                            const int q = landed - rbase;
#ifdef K5_NO_TMA
                            if (q >= kSlots) continue;
#endif
                            K5ACC(st_full, mbar_wait(sfull + q % kSlots, (uint32_t)((q / kSlots) & 1)))
                        }
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    const uint64_t a0 = sdesc(sl_base + ((r - rbase) % kSlots) * kSlotBytes + kHaloOff * 16,
                                              kHaloX * 16, 128);
                    const uint64_t b0 = sdesc(sw_base + blk * kC * 16, kW2Icg, 128);
                    K5ACC(st_issue, umma_row12(dcol, a0, b0, idesc, first ? 0u : 1u))
#ifdef K5_TRACE
                    if (t == 2 && lane == 0 && rstamp < 24) K5T(rstamp++);
#endif
                };

                if (nr == 3) {
                    row(y + 1, 0, d, kIdesc192, true);      // [acc_y | acc_y+1 | acc_y+2] = A_y+1 [W_dy2 | W_dy1 | W_dy0]
                    row(y, 1, d, kIdesc128, false);         // [acc_y | acc_y+1] += A_y [W_dy1 | W_dy0]
                    row(y + 2, 0, d + 64, kIdesc128, false);  // [acc_y+1 | acc_y+2] += A_y+2 [W_dy2 | W_dy1]
                    row(y - 1, 2, d, kIdesc, false);        // acc_y += A_y-1 W_dy0
                    row(y + 3, 0, d + 128, kIdesc, false);  // acc_y+2 += A_y+3 W_dy2
                } else if (nr == 2) {
                    row(y, 1, d, kIdesc128, true);          // [acc_y | acc_y+1] = A_y [W_dy1 | W_dy0]
                    row(y + 1, 0, d, kIdesc128, false);     // += A_y+1 [W_dy2 | W_dy1]
                    row(y - 1, 2, d, kIdesc, false);        // acc_y += A_y-1 W_dy0
                    row(y + 2, 0, d + 64, kIdesc, false);   // acc_y+1 += A_y+2 W_dy2
                } else {
                    row(y - 1, 2, d, kIdesc, true);
                    row(y, 1, d, kIdesc, false);
                    row(y + 1, 0, d, kIdesc, false);
                }
                umma_commit_e(afull + b);
#ifdef K5_TRACE
                if (t == 2 && lane == 0) K5T(24);
#endif
                if (lane == 0 && t < 8) {
                    K5T(2 + 2 * t);
                    K5V(32 + t, st_full);
                    K5V(40 + t, st_acc);
                    K5V(56 + t, st_issue);
                }
#ifndef K5_NO_SLOTCOMMIT  // (timing experiment with K5_NO_TMA)
                for (int r = y - 1; r < y - 1 + nr; ++r)  // rows y-1 .. y+nr-2: last read by this unit
                    umma_commit_e(sempty + (r - rbase) % kSlots);
#endif
#ifdef K5_TRACE
                if (t == 2 && lane == 0) K5T(25);
#endif
            }
        }
    } else {  // ---- epilogue warps 2..5
        const int quad = warp & 3;
        for (int t = 0; t < n_units; ++t) {
            const int y = y0 + R * t, b = t & 1, ub = t >> 1;
            const int nrows = min(R, y1 - y);
            mbar_wait(afull + b, (uint32_t)(ub & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int rr = 0; rr < nrows; ++rr) {
                const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * R * 64 + rr * 64);
                uint32_t r[64];
#ifdef K5_NO_LD  // timing experiment only: the accumulators are not read
                for (int i = 0; i < 64; ++i) r[i] = base + i;
#else
                LD16(base + 0, (r + 0));
                LD16(base + 16, (r + 16));
                LD16(base + 32, (r + 32));
                LD16(base + 48, (r + 48));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#endif
                if (rr == nrows - 1) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + b)) : "memory");
                }
                const int px = x0 + quad * 32 + lane;
                if (rr == 0 && warp == 2 && lane == 0 && t < 8) K5T(3 + 2 * t);  // accumulators read
#ifdef K5_NO_STORE  // timing experiment only: skip the activation stores
                if (px < 0) {
#else
                if (px < W) {
#endif
                    uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)(y + rr) * Wp + px);
                    const size_t gstride = (size_t)H * Wp;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        uint32_t pk[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const float lo = fmaxf(__uint_as_float(r[8 * q + 2 * h]), 0.f);
                            const float hi = fmaxf(__uint_as_float(r[8 * q + 2 * h + 1]), 0.f);
                            const __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, hi);
                            pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
                        }
                        dst[q * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                }
            }
            if (warp == 2 && lane == 0 && t < 8) K5T(50 + t);  // unit stored
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        K5T(31);
        K5V(49, k5_gtime());
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAccCols) : "memory");
}

// Rolling-accumulator variant of the 64->64 layer (k_conv64_roll, the default).  The issue path of
// the row-unit kernels is the bottleneck, not the tensor pipe: a UMMA costs the issuing thread ~45-58
// cycles whatever its N (tools/micro/umma_rate.cu: 44.7 cycles per M = 128 UMMA at N = 16..64), the
// N = 64 UMMAs of a unit's first and last halo rows run at 48 cycles for 32 cycles of math, and the
// four commits and waits at every unit boundary drain the pipe (tools/micro/k5_trace3.cu: 4,750 cycles
// per row triple against 3,835 for the same 60 UMMAs alone).  Here every halo row r is ONE run of
// N = 192 UMMAs against [W_dy2 | W_dy1 | W_dy0] into the accumulators of output rows r-1, r, r+1,
// which sit side by side in TMEM: output row y owns the 64 columns of slot (y - y0) mod 8, so the
// three accumulators of a halo row are contiguous except where the window wraps (2 rows in 8: split
// into N = 128 + N = 64).  Row r+1's accumulator starts with this halo row, so the first of the 12
// (dx, K-step) UMMAs is issued as N = 128 accumulating + N = 64 overwriting and the other 11 as
// N = 192: 13 UMMAs and 1,168 tensor cycles per output row (1,152 = pure math) instead of 20 UMMAs
// and 1,280.  One commit per halo row (rowdone) tells the epilogue that output row r-1 is complete
// and the TMA producer that the halo slot is free; the epilogue drains one row at a time.
__device__ __forceinline__ void umma_row13(uint32_t d_tmem, uint64_t a0, uint64_t b0)
{
    static_assert(kHaloX == 144 && kW2Dx == 24576 && kW2Icg == 3072, "offsets below are hard-coded");
    asm volatile(
        "{\n.reg .pred e, f, t;\n.reg .b64 a, b;\n.reg .b32 d2;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.eq.b32 t, 1, 1;\nsetp.ne.b32 f, 1, 1;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, t;\n"          // rows r-1, r: += A [W_dy2 | W_dy1]
        "add.u32 d2, %0, 128;\nadd.s64 b, %2, 128;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [d2], %1, b, %4, f;\n"           // row r+1: = A W_dy0
        "add.s64 a, %1, 288;\nadd.s64 b, %2, 384;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 576;\nadd.s64 b, %2, 768;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 864;\nadd.s64 b, %2, 1152;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 1;\nadd.s64 b, %2, 1536;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 289;\nadd.s64 b, %2, 1920;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 577;\nadd.s64 b, %2, 2304;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 865;\nadd.s64 b, %2, 2688;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 2;\nadd.s64 b, %2, 3072;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 290;\nadd.s64 b, %2, 3456;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 578;\nadd.s64 b, %2, 3840;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "add.s64 a, %1, 866;\nadd.s64 b, %2, 4224;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(kIdesc128), "r"(kIdesc), "r"(kIdesc192)
        : "memory");
}
// the 11 (dx, K-step) UMMAs after the first, all accumulating (generic rows: one call per run of
// contiguous accumulators)
__device__ __forceinline__ void umma_row11(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc)
{
    asm volatile(
        "{\n.reg .pred e, t;\n.reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.eq.b32 t, 1, 1;\n"
        "add.s64 a, %1, 288;\nadd.s64 b, %2, 384;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 576;\nadd.s64 b, %2, 768;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 864;\nadd.s64 b, %2, 1152;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 1;\nadd.s64 b, %2, 1536;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 289;\nadd.s64 b, %2, 1920;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 577;\nadd.s64 b, %2, 2304;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 865;\nadd.s64 b, %2, 2688;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 2;\nadd.s64 b, %2, 3072;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 290;\nadd.s64 b, %2, 3456;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 578;\nadd.s64 b, %2, 3840;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "add.s64 a, %1, 866;\nadd.s64 b, %2, 4224;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(idesc)
        : "memory");
}

// a wrapping halo row as one asm block: run A (12 UMMAs into dA) interleaved with run B (into dB: the first
// UMMA with its own descriptor and accumulate flag, the other 11 accumulating with idB_rest) and, if hasC,
// one overwriting N = 64 UMMA into dC next to the first pair
__device__ __forceinline__ void umma_row_wrap(uint64_t a0, uint32_t dA, uint64_t bA, uint32_t idA, uint32_t dB, uint64_t bB,
                                              uint32_t idB_first, uint32_t idB_rest, uint32_t accB_first, uint32_t dC,
                                              uint64_t bC, uint32_t hasC)
{
    asm volatile(
        "{\n.reg .pred e, ec, pb, t, f;\n.reg .b64 a, b, c;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.eq.b32 t, 1, 1;\nsetp.ne.b32 f, 1, 1;\nsetp.ne.b32 pb, %8, 0;\n"
        "setp.ne.b32 ec, %11, 0;\nand.pred ec, ec, e;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %0, %2, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%4], %0, %5, %6, pb;\n"
        "@ec tcgen05.mma.cta_group::1.kind::f16 [%9], %0, %10, %12, f;\n"
#define WR(ao, bo)                                                                                      \
    "add.s64 a, %0, " #ao ";\nadd.s64 b, %2, " #bo ";\nadd.s64 c, %5, " #bo ";\n"                     \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%1], a, b, %3, t;\n@e tcgen05.mma.cta_group::1.kind::f16 [%4], a, c, %7, t;\n"
        WR(288, 384) WR(576, 768) WR(864, 1152) WR(1, 1536) WR(289, 1920) WR(577, 2304) WR(865, 2688) WR(2, 3072)
        WR(290, 3456) WR(578, 3840) WR(866, 4224)
#undef WR
        "}\n"
        ::"l"(a0), "r"(dA), "l"(bA), "r"(idA), "r"(dB), "l"(bB), "r"(idB_first), "r"(idB_rest), "r"(accB_first), "r"(dC),
          "l"(bC), "r"(hasC), "r"(kIdesc)
        : "memory");
}

#ifndef K5_FIRST_ROWS
#define K5_FIRST_ROWS 2  // halo rows issued before the producer waits for the first one to land (0: no wait; 0.2090 -> 0.2070 ms)
#endif
constexpr int kRollAcc = 8;  // accumulator slots of 64 fp32 columns: all 512 TMEM columns

// kSeq: all n_layers middle layers in one cooperative launch.  Every CTA keeps its (strip, row run); the
// halo ring, the accumulator slots and every mbarrier phase simply run on from layer to layer.  Layer l
// reads act[l % 2] (map0 / map1) and writes act[(l + 1) % 2].  Between layers a grid-wide arrive / wait on
// one counter: after a layer's last row the epilogue warps fence their stores and one thread adds 1
// (release); the producer waits for (epoch x (n_layers - 1) + l) x CTAs arrivals (acquire), then a proxy
// fence orders the TMA reads behind the other CTAs' generic-proxy stores.  The same wait covers the
// write-after-read hazard of the ping-pong buffers (every CTA has finished reading layer l - 1's input
// before anyone writes layer l's output over it).  The next layer's weights are copied in as soon as the
// layer's last UMMA has completed, i.e. during the wait.
__device__ unsigned g_k5_sync_timeout;  // set if a grid-wide wait ever gave up (never, unless a CTA died)

template <bool kSeq>
__global__ void __launch_bounds__(192, 1) k_conv64_roll(const __grid_constant__ CUtensorMap map0,
                                                        const __grid_constant__ CUtensorMap map1,
                                                        const __nv_bfloat16* __restrict__ wts, __nv_bfloat16* out0,
                                                        __nv_bfloat16* out1, int H, int W, int Wp, int rows_per_cta,
                                                        int n_layers, unsigned* sync_ctr, unsigned sync_base)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;
    unsigned char* slots = sm + kWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;
    uint64_t* sfull = bars + 1;             // [kSlots] halo row landed
    uint64_t* rowdone = sfull + kSlots;     // [kSlots] the halo row's UMMAs have completed
    uint64_t* aempty = rowdone + kSlots;    // [kRollAcc] accumulator slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kRollAcc);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef K5_TRACE
    __shared__ unsigned life_idx;
    if (tid == 0) {
        K5T(0);
        K5V(48, k5_gtime());
        life_idx = atomicAdd(&g_k5_life_n, 1u) % 4096u;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_k5_life[life_idx][0] = smid;
        g_k5_life[life_idx][1] = k5_gtime();
    }
#endif
    if constexpr (!kSeq) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips;
    const int x0 = strip * kTileX;
    const int y0 = (blockIdx.x / strips) * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    if (y0 >= H) return;  // (never in a kSeq launch: the grid is exactly the CTAs that own rows)
    const int nrows = y1 - y0, nq = nrows + 2;  // output rows and halo rows per layer
    const int L = kSeq ? n_layers : 1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kRollAcc * 64)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(rowdone + i, 1);
        }
        for (int i = 0; i < kRollAcc; ++i) mbar_init(aempty + i, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;  // halo row r of a layer has index q = r - rbase; ring index Q = l nq + q

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            for (int l = 0; l < L; ++l) {
                if (l > 0) {  // the weights buffer is free once the previous layer's last halo row is done
                    const int Ql = l * nq - 1;
                    mbar_wait(rowdone + Ql % kSlots, (uint32_t)((Ql / kSlots) & 1));
                }
                mbar_expect(wbar, kWBytes);
                bulk_copy(sw, wts + (size_t)l * 9 * kC * kC, kWBytes, wbar);
                if (l == 0) {
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    K5T(30);
#ifdef K5_TRACE
                    g_k5_life[life_idx][2] = k5_gtime();
#endif
                } else {
                    // every CTA has stored (and fenced) layer l - 1
                    const unsigned target = sync_base + (unsigned)l * gridDim.x;
                    unsigned seen, spins = 0;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(sync_ctr) : "memory");
                        if ((int)(seen - target) >= 0) break;
                        if (++spins > (1u << 26)) {  // seconds: a CTA died; give up loudly rather than hang
                            g_k5_sync_timeout = 1u;
                            __trap();
                        }
                    } while (true);
                    asm volatile("fence.proxy.async;" ::: "memory");
                }
                const CUtensorMap* map = (l & 1) ? &map1 : &map0;
                for (int q = 0; q < nq; ++q) {
                    const int Q = l * nq + q, s = Q % kSlots, u = Q / kSlots;
                    if (u >= 1) mbar_wait(rowdone + s, (uint32_t)((u - 1) & 1));
                    mbar_expect(sfull + s, kSlotBytes);
                    tma_row(slots + s * kSlotBytes, map, x0 / 8 - 1, rbase + q, sfull + s);
#if K5_FIRST_ROWS > 0
                    // every CTA starts its layer at the same moment: let the first halo rows of all CTAs through
                    // L2 before the rest of the ring (8 rows x 148 CTAs = 22 MB at once) queues up behind them
                    if (!kSeq && q == K5_FIRST_ROWS - 1) mbar_wait(sfull, 0u);
#endif
                }
            }
        }
    } else if (warp == 1) {  // ---- MMA issuer (whole warp, one elected lane issues)
        const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
        [[maybe_unused]] long long st_full = 0, st_acc = 0, st_issue = 0, st_commit = 0, st_wrap = 0;
        for (int l = 0; l < L; ++l) {
            mbar_wait(wbar, (uint32_t)(l & 1));
            if (lane == 0 && l == 0) K5T(1);
            for (int q = 0; q < nq; ++q) {
                const int r = rbase + q;
                const int Q = l * nq + q, s = Q % kSlots;
                // accumulators fed by this halo row: output rows r-1 (W_dy2), r (W_dy1), r+1 (W_dy0); output
                // row i of layer l has the running index I = l nrows + i and lives in slot I mod 8
                const bool v0 = r - 1 >= y0, v1 = r >= y0 && r < y1, v2 = r + 1 < y1;
                const int I2 = l * nrows + q;  // running index of output row r + 1
                if (v2 && I2 >= kRollAcc) {    // its slot: drained of the row that had it before?
                    K5ACC(st_acc, mbar_wait(aempty + (I2 % kRollAcc), (uint32_t)((I2 / kRollAcc - 1) & 1)))
                }
                K5ACC(st_full, mbar_wait(sfull + s, (uint32_t)((Q / kSlots) & 1)))
                if (lane == 0 && Q == 0) K5T(31);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t abase = sl_base + s * kSlotBytes + kHaloOff * 16;
                const uint64_t a0 = sdesc(abase, kHaloX * 16, 128);
                const int s0 = (I2 + 2 * kRollAcc - 2) % kRollAcc;  // slot of output row r-1; r: s0+1, r+1: s0+2 (mod 8)
                // B = [W_dy2 | W_dy1 | W_dy0] from block k on; accumulator of block k in slot (s0 + k) mod 8
                auto bd = [&](int k) { return sdesc(sw_base + k * kC * 16, kW2Icg, 128); };
                auto dc = [&](int k) { return tmem + (uint32_t)(((s0 + k) % kRollAcc) * 64); };
                if (v0 && v1 && v2) {
                    if (s0 + 2 < kRollAcc) {
                        K5ACC(st_issue, umma_row13(dc(0), a0, bd(0)))
                    } else if (s0 + 1 < kRollAcc) {  // slots 6, 7 | 0
                        K5ACC(st_wrap, umma_row_wrap(a0, dc(0), bd(0), kIdesc128, dc(2), bd(2), kIdesc, kIdesc, 0u, 0u, 0ull, 0u))
                    } else {  // slots 7 | 0, 1: rows r, r+1 share all but the first UMMA (row r+1's overwrites)
                        K5ACC(st_wrap, umma_row_wrap(a0, dc(0), bd(0), kIdesc, dc(1), bd(1), kIdesc, kIdesc128, 1u, dc(2), bd(2), 1u))
                    }
                } else if (v1 && v2 && !v0 && (s0 + 1) % kRollAcc + 1 < kRollAcc) {  // the CTA's first image row
                    umma_e(dc(1), a0, bd(1), kIdesc, 1u);
                    umma_e(dc(2), a0, bd(2), kIdesc, 0u);
                    umma_row11(dc(1), a0, bd(1), kIdesc128);
                } else if (v0 && v1 && !v2 && s0 + 1 < kRollAcc) {  // the CTA's last image row
                    umma_row12(dc(0), a0, bd(0), kIdesc128, 1u);
                } else {  // top and bottom halo rows, short CTAs, wrapping edge rows: one N = 64 run per accumulator
                    if (v0) umma_row12(dc(0), a0, bd(0), kIdesc, 1u);
                    if (v1) umma_row12(dc(1), a0, bd(1), kIdesc, 1u);
                    if (v2) umma_row12(dc(2), a0, bd(2), kIdesc, 0u);
                }
                K5ACC(st_commit, umma_commit_e(rowdone + s))
                if (lane == 0 && Q < 16) K5T(2 + Q);
                if (lane == 0 && Q < 14) K5V(50 + Q, st_full + st_acc);
            }
        }
        if (lane == 0) {
            K5V(18, st_full);
            K5V(19, st_acc);
            K5V(20, st_issue);
            K5V(21, st_commit);
            K5V(22, st_wrap);
        }
    } else {  // ---- epilogue warps 2..5: output row y is complete once halo row y+1 is done
        const int quad = warp & 3;
        for (int l = 0; l < L; ++l) {
            __nv_bfloat16* out = (l & 1) ? out1 : out0;
            for (int y = y0; y < y1; ++y) {
                const int Q = l * nq + (y + 1 - rbase), a = (l * nrows + (y - y0)) % kRollAcc;
                mbar_wait(rowdone + Q % kSlots, (uint32_t)((Q / kSlots) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * 64);
                uint32_t r[64];
                LD16(base + 0, (r + 0));
                LD16(base + 16, (r + 16));
                LD16(base + 32, (r + 32));
                LD16(base + 48, (r + 48));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (warp == 2 && lane == 0 && l == 0 && y - y0 < 14) K5T(32 + y - y0);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + a)) : "memory");
                const int px = x0 + quad * 32 + lane;
                if (px < W) {
                    uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)y * Wp + px);
                    const size_t gstride = (size_t)H * Wp;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        uint32_t pk[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const float lo = fmaxf(__uint_as_float(r[8 * g + 2 * h]), 0.f);
                            const float hi = fmaxf(__uint_as_float(r[8 * g + 2 * h + 1]), 0.f);
                            const __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, hi);
                            pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
                        }
                        dst[g * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                }
            }
            if (kSeq && l + 1 < L) {  // this CTA's share of layer l is stored: fence, then one arrival
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tid == 64) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(sync_ctr) : "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
#ifdef K5_TRACE
    if (tid == 0) {
        K5V(49, k5_gtime());
        g_k5_life[life_idx][3] = k5_gtime();
    }
#endif
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kRollAcc * 64) : "memory");
}

// Pipelined persistent variant (k_conv64_pipe, MACE_K5_SEQ=2): all middle layers in one cooperative launch
// WITHOUT a grid-wide wait between layers.  In odd layers every CTA's row run is shifted up by half a run
// (run j owns rows [per j - per/2, per (j+1) - per/2); the first run is half as long, the last takes the rest),
// and every CTA sweeps its run top to bottom.  The rows a CTA needs first in layer l+1 (and their neighbours in
// the adjacent strips) were then written in the MIDDLE of layer l, half a layer (~4 us) earlier, and the rows
// written last in layer l are needed last in layer l+1: no CTA ever waits for a row that has only just been
// stored, so the layers run back to back.  Read-after-write: every epilogue warp publishes, after each output
// row it has stored and fenced, its running row count in flags[cta][warp] (release); before the TMA producer
// loads halo row r of layer l+1 it acquires the counts of the (up to three strips') owners of row r in layer l,
// then orders the async-proxy read behind them (fence.proxy.async).  Write-after-read on the ping-pong buffers
// follows from the same waits: row r of layer l+1 is stored after rows r-1..r+1 of layer l (strips s-1..s+1)
// were complete, and computing those is what read the rows of the buffer that row r overwrites.
struct RowRun {
    int y0, y1;
};
__device__ __forceinline__ RowRun pipe_run(int j, int odd, int per, int nyc, int H)
{
    const int half = odd ? per / 2 : 0;
    RowRun r;
    r.y0 = max(0, per * j - half);
    r.y1 = j == nyc - 1 ? H : per * (j + 1) - half;
    return r;
}
__device__ __forceinline__ int pipe_owner(int row, int odd, int per, int nyc)
{
    return min(nyc - 1, (row + (odd ? per / 2 : 0)) / per);
}
// rows run j has completed before layer l (layers 0, 2, .. are even)
__device__ __forceinline__ int pipe_cum(int j, int l, int per, int nyc, int H)
{
    const RowRun e = pipe_run(j, 0, per, nyc, H), o = pipe_run(j, 1, per, nyc, H);
    return ((l + 1) / 2) * (e.y1 - e.y0) + (l / 2) * (o.y1 - o.y0);
}

constexpr int kPSlots = 4;                                            // halo ring of k_conv64_pipe
constexpr int kPSmem = 2 * kWBytes + kPSlots * kSlotBytes + 1024;     // two weight buffers + ring: 222,208 B
constexpr int kPThreads = 320;                                        // producer, issuer, 2 x 4 epilogue warps

__global__ void __launch_bounds__(kPThreads, 1) k_conv64_pipe(const __grid_constant__ CUtensorMap map0,
                                                              const __grid_constant__ CUtensorMap map1,
                                                              const __nv_bfloat16* __restrict__ wts, __nv_bfloat16* out0,
                                                              __nv_bfloat16* out1, int H, int W, int Wp, int per,
                                                              int n_layers, unsigned* flags, unsigned flag_base)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;                   // weights of layer l in buffer l & 1
    unsigned char* slots = sm + 2 * kWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kPSlots * kSlotBytes);
    // rowdone barriers in a ring of 16: without a grid-wide wait the MMA issuer can be a layer boundary (two extra
    // halo rows) ahead of the epilogue, so with a short ring a parity wait could miss a whole phase
    constexpr int kRD = 16;
    uint64_t* wbar = bars;                  // [2]
    uint64_t* sfull = bars + 2;             // [kPSlots]
    uint64_t* rowdone = sfull + kPSlots;    // [kRD]
    uint64_t* aempty = rowdone + kRD;       // [kRollAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kRollAcc);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips, jrun = blockIdx.x / strips;
    const int nyc = gridDim.x / strips;
    const int x0 = strip * kTileX;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kRollAcc * 64)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        mbar_init(wbar + 1, 1);
        for (int i = 0; i < kPSlots; ++i) mbar_init(sfull + i, 1);
        for (int i = 0; i < kRD; ++i) mbar_init(rowdone + i, 1);
        for (int i = 0; i < kRollAcc; ++i) mbar_init(aempty + i, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ---- TMA producer (whole warp: lanes 0..11 watch the owners' flags, lane 0 copies)
        int Qb = 0;   // halo rows before this layer
        // lane 4 t + w watches TMEM quarter w of the owners in strip (strip - 1 + t); a run's rows alternate between
        // its two epilogue groups (running row index mod 2), each with its own count
        const int ft = lane >> 2, fw = lane & 3, fstrip = strip - 1 + ft;
        const bool watcher = lane < 12 && fstrip >= 0 && fstrip < strips;
        unsigned seen[2] = {flag_base, flag_base};
        int seen_owner = -1;
        if (lane == 0) {
            for (int l = 0; l < 2 && l < n_layers; ++l) {
                mbar_expect(wbar + l, kWBytes);
                bulk_copy(sw + l * kWBytes, wts + (size_t)l * 9 * kC * kC, kWBytes, wbar + l);
            }
        }
        for (int l = 0; l < n_layers; ++l) {
            const RowRun rr = pipe_run(jrun, l & 1, per, nyc, H);
            const int nq = rr.y1 - rr.y0 + 2;
            const CUtensorMap* map = (l & 1) ? &map1 : &map0;
            // owner of the current halo row in layer l - 1: its run and the rows it had completed before that layer
            int jo = -1, oy0 = 0, oy1 = -1, ocum = 0;
            for (int q = 0; q < nq; ++q) {
                const int r = rr.y0 - 1 + q;
#ifdef K5P_NOPOLL  // (timing experiment)
                if (false) {
#else
                if (l > 0 && r >= 0 && r < H) {  // row r of layer l - 1: stored and visible?
#endif
                    if (r >= oy1 || jo < 0) {
                        jo = pipe_owner(r, (l - 1) & 1, per, nyc);
                        const RowRun ro = pipe_run(jo, (l - 1) & 1, per, nyc, H);
                        oy0 = ro.y0;
                        oy1 = ro.y1;
                        ocum = pipe_cum(jo, l - 1, per, nyc, H);
                    }
                    bool polled = false;
                    if (watcher) {
                        const int I = ocum + r - oy0;  // the row's running index in its owner
                        const unsigned need = flag_base + (unsigned)(I + 1);
                        if (seen_owner != jo) {
                            seen[0] = seen[1] = flag_base;
                            seen_owner = jo;
                        }
                        if ((int)(seen[I & 1] - need) < 0) {
                            const unsigned* f = flags + (((size_t)(jo * strips + fstrip) * 4 + fw) * 2 + (I & 1));
                            unsigned v, spins = 0;
                            do {
                                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                                if ((int)(v - need) >= 0) break;
                                if (++spins > (1u << 22)) {  // seconds: give up loudly rather than hang
                                    g_k5_sync_timeout = 2u;
                                    __trap();
                                }
                            } while (true);
                            seen[I & 1] = v;
                            polled = true;
                        }
                    }
                    if (__any_sync(0xffffffffu, polled)) asm volatile("fence.proxy.async;" ::: "memory");
                }
                if (lane == 0) {
                    const int Q = Qb + q, s = Q % kPSlots;
                    if (Q >= kPSlots) mbar_wait(rowdone + (Q - kPSlots) % kRD, (uint32_t)(((Q - kPSlots) / kRD) & 1));
                    mbar_expect(sfull + s, kSlotBytes);
                    tma_row(slots + s * kSlotBytes, map, x0 / 8 - 1, r, sfull + s);
                    // the next layer's weights into the other buffer, once the previous layer (its last user) is done
                    if (q == min(kPSlots - 1, nq - 1) && l >= 1 && l + 1 < n_layers) {
                        mbar_wait(rowdone + (Qb - 1) % kRD, (uint32_t)(((Qb - 1) / kRD) & 1));
                        mbar_expect(wbar + ((l + 1) & 1), kWBytes);
                        bulk_copy(sw + ((l + 1) & 1) * kWBytes, wts + (size_t)(l + 1) * 9 * kC * kC, kWBytes,
                                  wbar + ((l + 1) & 1));
                    }
                }
                __syncwarp();
            }
            Qb += nq;
        }
    } else if (warp == 1) {  // ---- MMA issuer (whole warp, one elected lane issues)
        const uint32_t sl_base = s_u32(slots);
        int Qb = 0, Ib = 0;
        for (int l = 0; l < n_layers; ++l) {
            const RowRun rr = pipe_run(jrun, l & 1, per, nyc, H);
            const int y0 = rr.y0, y1 = rr.y1, nq = y1 - y0 + 2;
            const uint32_t sw_base = s_u32(sw + (l & 1) * kWBytes);
            mbar_wait(wbar + (l & 1), (uint32_t)((l >> 1) & 1));
            for (int q = 0; q < nq; ++q) {
                const int r = y0 - 1 + q;
                const int Q = Qb + q, s = Q % kPSlots;
                const bool v0 = r - 1 >= y0, v1 = r >= y0 && r < y1, v2 = r + 1 < y1;
                const int I2 = Ib + q;  // running index of output row r + 1
                if (v2 && I2 >= kRollAcc) mbar_wait(aempty + (I2 % kRollAcc), (uint32_t)((I2 / kRollAcc - 1) & 1));
                mbar_wait(sfull + s, (uint32_t)((Q / kPSlots) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t a0 = sdesc(sl_base + s * kSlotBytes + kHaloOff * 16, kHaloX * 16, 128);
                const int s0 = (I2 + 2 * kRollAcc - 2) % kRollAcc;
                auto bd = [&](int k) { return sdesc(sw_base + k * kC * 16, kW2Icg, 128); };
                auto dc = [&](int k) { return tmem + (uint32_t)(((s0 + k) % kRollAcc) * 64); };
                if (v0 && v1 && v2) {
                    if (s0 + 2 < kRollAcc) {
                        umma_row13(dc(0), a0, bd(0));
                    } else if (s0 + 1 < kRollAcc) {
                        umma_row_wrap(a0, dc(0), bd(0), kIdesc128, dc(2), bd(2), kIdesc, kIdesc, 0u, 0u, 0ull, 0u);
                    } else {
                        umma_row_wrap(a0, dc(0), bd(0), kIdesc, dc(1), bd(1), kIdesc, kIdesc128, 1u, dc(2), bd(2), 1u);
                    }
                } else if (v1 && v2 && !v0 && (s0 + 1) % kRollAcc + 1 < kRollAcc) {
                    umma_e(dc(1), a0, bd(1), kIdesc, 1u);
                    umma_e(dc(2), a0, bd(2), kIdesc, 0u);
                    umma_row11(dc(1), a0, bd(1), kIdesc128);
                } else if (v0 && v1 && !v2 && s0 + 1 < kRollAcc) {
                    umma_row12(dc(0), a0, bd(0), kIdesc128, 1u);
                } else {
                    if (v0) umma_row12(dc(0), a0, bd(0), kIdesc, 1u);
                    if (v1) umma_row12(dc(1), a0, bd(1), kIdesc, 1u);
                    if (v2) umma_row12(dc(2), a0, bd(2), kIdesc, 0u);
                }
                umma_commit_e(rowdone + Q % kRD);
            }
            Qb += nq;
            Ib += y1 - y0;
        }
    } else {  // ---- epilogue warps 2..9: two groups of four (TMEM quarter = warp mod 4), alternating output rows, so
              // that the fence behind every row's stores has two row times to complete
        const int quad = warp & 3, grp = (warp - 2) >> 2;
        unsigned* myflag = flags + (((size_t)blockIdx.x * 4 + quad) * 2 + grp);
        int Qb = 0, Ib = 0;
        for (int l = 0; l < n_layers; ++l) {
            const RowRun rr = pipe_run(jrun, l & 1, per, nyc, H);
            const int y0 = rr.y0, y1 = rr.y1;
            __nv_bfloat16* out = (l & 1) ? out1 : out0;
            for (int y = y0; y < y1; ++y) {
                const int I = Ib + (y - y0);
                if ((I & 1) != grp) continue;
                const int Q = Qb + (y - y0 + 2), a = I % kRollAcc;
                mbar_wait(rowdone + Q % kRD, (uint32_t)((Q / kRD) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * 64);
                uint32_t r[64];
                LD16(base + 0, (r + 0));
                LD16(base + 16, (r + 16));
                LD16(base + 32, (r + 32));
                LD16(base + 48, (r + 48));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + a)) : "memory");
                const int px = x0 + quad * 32 + lane;
                if (px < W) {
                    uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)y * Wp + px);
                    const size_t gstride = (size_t)H * Wp;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        uint32_t pk[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const float lo = fmaxf(__uint_as_float(r[8 * g + 2 * h]), 0.f);
                            const float hi = fmaxf(__uint_as_float(r[8 * g + 2 * h + 1]), 0.f);
                            const __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, hi);
                            pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
                        }
                        dst[g * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                }
                if (l + 1 < n_layers) {  // publish: this warp's part of its rows .. y is stored and visible
#ifndef K5P_NOFENCE  // (timing experiment)
                    __threadfence();
#endif
                    __syncwarp();
                    if (lane == 0) {
                        const unsigned v = flag_base + (unsigned)(I + 1);
                        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(myflag), "r"(v) : "memory");
                    }
                }
            }
            Qb += y1 - y0 + 2;
            Ib += y1 - y0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kRollAcc * 64) : "memory");
}

// All 15 middle layers in ONE persistent launch (k_conv64_seq): every CTA keeps its (strip, row run)
// for the whole stack, its TMEM allocation and barriers live across layers, and the halo-row ring,
// accumulator pair ring and mbarrier phases simply continue from layer to layer.  Layer l reads
// act[l % 2] and writes act[(l + 1) % 2].  Between layers a CTA waits only for its 3 x 3
// neighbourhood: after its epilogue warps have stored a layer's rows (and fenced them), one thread
// publishes flags[cta] = 16 epoch + l + 1 (release); before loading halo rows for layer l the TMA
// thread acquires flags >= 16 epoch + l of itself and its neighbours, then a proxy fence orders the
// TMA (async proxy) reads after those generic-proxy writes.  Because a neighbour's flag for layer l - 1
// also means it has finished READING act[(l - 1) % 2] = the buffer layer l overwrites, the same wait
// covers the write-after-read hazard.  The next layer's 72 KB of weights are copied in as soon as
// the MMA issuer has committed the layer's last UMMA (wfree).  Launched cooperatively (all CTAs
// co-resident: one per SM), so the spin-waits cannot deadlock.  Measured SLOWER than 15 launches with
// programmatic dependent launch (0.333 vs 0.277 ms per 512^2 denoise on B200), so it is an option
// (MACE_K5_SEQ=1), bit-identical to the default (tests/test_gpu_cnn.py); DESIGN.md §6.
#ifdef K5SEQ_TRACE  // profiling builds only: per-CTA, per-layer %globaltimer stamps of k_conv64_seq
// [cta][layer][0 weights free seen, 1 neighbour flags passed, 2 weights landed (MMA), 3 first unit
// issued, 4 last unit issued, 5 layer published]
__device__ unsigned long long g_k5seq[148][16][6];
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define K5S(l, i) (blockIdx.x < 148 && (l) < 16 ? (void)(g_k5seq[blockIdx.x][(l)][(i)] = gtimer()) : (void)0)
#else
#define K5S(l, i) ((void)0)
#endif

__device__ __forceinline__ void flag_wait_ge(const int* f, int v)
{
    int x;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
        if (x >= v) break;
    }
}

__global__ void __launch_bounds__(192, 1) k_conv64_seq(const __grid_constant__ CUtensorMap map0,
                                                       const __grid_constant__ CUtensorMap map1,
                                                       const __nv_bfloat16* __restrict__ wts, __nv_bfloat16* act0,
                                                       __nv_bfloat16* act1, int H, int W, int Wp, int rows_per_cta,
                                                       int n_layers, int* flags, int epoch)
{
    constexpr int R = 2;
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;
    unsigned char* slots = sm + kWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;
    uint64_t* sfull = bars + 1;
    uint64_t* sempty = sfull + kSlots;
    uint64_t* afull = sempty + kSlots;  // [2] accumulator pair ready
    uint64_t* aempty = afull + 2;       // [2] accumulator pair drained
    uint64_t* wfree = aempty + 2;       // the layer's last UMMA completed: weights may be replaced
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfree + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips, rb = blockIdx.x / strips;
    const int x0 = strip * kTileX;
    const int y0 = rb * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    const int n_rb = (H + rows_per_cta - 1) / rows_per_cta;
    if (y0 >= H) return;  // never: the grid is exactly strips x n_rb
    const int n_units = (y1 - y0 + R - 1) / R;
    const int rows_l = y1 - y0 + 2;  // halo rows per layer (y0 - 1 .. y1)
    constexpr int kAccCols = 256;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kAccCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        mbar_init(wfree, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(sempty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(afull + i, 1);
            mbar_init(aempty + i, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            long q0 = 0;
            for (int l = 0; l < n_layers; ++l) {
                if (l > 0) mbar_wait(wfree, (uint32_t)((l - 1) & 1));
                K5S(l, 0);
                mbar_expect(wbar, kWBytes);
                bulk_copy(sw, wts + (size_t)l * 9 * kC * kC, kWBytes, wbar);
                if (l > 0) {  // the neighbourhood's layer l - 1 is written (and its layer l - 1 reads are done)
                    const int want = 16 * epoch + l;
                    for (int dr = -1; dr <= 1; ++dr)
                        for (int dc = -1; dc <= 1; ++dc) {
                            const int r2 = rb + dr, c2 = strip + dc;
                            if (r2 >= 0 && r2 < n_rb && c2 >= 0 && c2 < strips) flag_wait_ge(flags + r2 * strips + c2, want);
                        }
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                K5S(l, 1);
                const CUtensorMap* m = (l & 1) ? &map1 : &map0;
                for (int r = y0 - 1; r <= y1; ++r) {
                    const long q = q0 + (r - rbase);
                    const int s = (int)(q % kSlots);
                    const long u = q / kSlots;
                    if (u >= 1) mbar_wait(sempty + s, (uint32_t)((u - 1) & 1));
                    mbar_expect(sfull + s, kSlotBytes);
                    tma_row(slots + s * kSlotBytes, m, x0 / 8 - 1, r, sfull + s);
                }
                q0 += rows_l;
            }
        }
    } else if (warp == 1) {  // ---- MMA issuer (whole warp, one elected lane issues)
        const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
        long q0 = 0;
        int tg = 0;  // accumulator-pair units issued so far (all layers)
        for (int l = 0; l < n_layers; ++l) {
            mbar_wait(wbar, (uint32_t)(l & 1));
            if (lane == 0) K5S(l, 2);
            int landed = y0 - 2;
            int y_last = y0, nr_last = 0;
            for (int t = 0; t < n_units; ++t, ++tg) {
                const int y = y0 + R * t, b = tg & 1, ub = tg >> 1;
                const int nr = min(R, y1 - y);
                if (ub >= 1) {
                    mbar_wait(aempty + b, (uint32_t)((ub - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                const uint32_t d = tmem + (uint32_t)(b * R * 64);
                auto row = [&](int r, int blk, uint32_t dcol, uint32_t idesc, bool first) {
                    if (r > landed) {
                        while (landed < r) {
                            ++landed;
                            const long q = q0 + (landed - rbase);
                            mbar_wait(sfull + q % kSlots, (uint32_t)((q / kSlots) & 1));
                        }
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    const long q = q0 + (r - rbase);
                    const uint64_t a0 = sdesc(sl_base + (uint32_t)(q % kSlots) * kSlotBytes + kHaloOff * 16, kHaloX * 16, 128);
                    const uint64_t b0 = sdesc(sw_base + blk * kC * 16, kW2Icg, 128);
                    umma_row12(dcol, a0, b0, idesc, first ? 0u : 1u);
                };
                if (nr == 2) {
                    row(y, 1, d, kIdesc128, true);
                    row(y + 1, 0, d, kIdesc128, false);
                    row(y - 1, 2, d, kIdesc, false);
                    row(y + 2, 0, d + 64, kIdesc, false);
                } else {
                    row(y - 1, 2, d, kIdesc, true);
                    row(y, 1, d, kIdesc, false);
                    row(y + 1, 0, d, kIdesc, false);
                }
                umma_commit_e(afull + b);
                for (int r = y - 1; r < y - 1 + nr; ++r) umma_commit_e(sempty + (q0 + r - rbase) % kSlots);
                if (lane == 0 && t == 0) K5S(l, 3);
                if (lane == 0 && t == n_units - 1) K5S(l, 4);
                y_last = y;
                nr_last = nr;
            }
            // rows never read again in this layer (the last unit's bottom halo) go back to the ring
            for (int r = y_last - 1 + nr_last; r <= y1; ++r) umma_commit_e(sempty + (q0 + r - rbase) % kSlots);
            umma_commit_e(wfree);
            q0 += rows_l;
        }
    } else {  // ---- epilogue warps 2..5
        const int quad = warp & 3;
        int tg = 0;
        for (int l = 0; l < n_layers; ++l) {
            __nv_bfloat16* out = (l & 1) ? act0 : act1;
            for (int t = 0; t < n_units; ++t, ++tg) {
                const int y = y0 + R * t, b = tg & 1, ub = tg >> 1;
                const int nrows = min(R, y1 - y);
                mbar_wait(afull + b, (uint32_t)(ub & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int rr = 0; rr < nrows; ++rr) {
                    const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * R * 64 + rr * 64);
                    uint32_t r[64];
                    LD16(base + 0, (r + 0));
                    LD16(base + 16, (r + 16));
                    LD16(base + 32, (r + 32));
                    LD16(base + 48, (r + 48));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (rr == nrows - 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + b)) : "memory");
                    }
                    const int px = x0 + quad * 32 + lane;
                    if (px < W) {
                        uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)(y + rr) * Wp + px);
                        const size_t gstride = (size_t)H * Wp;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            uint32_t pk[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const float lo = fmaxf(__uint_as_float(r[8 * q + 2 * h]), 0.f);
                                const float hi = fmaxf(__uint_as_float(r[8 * q + 2 * h + 1]), 0.f);
                                const __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, hi);
                                pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
                            }
                            dst[q * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        }
                    }
                }
            }
            // publish the layer: every epilogue thread's stores, then one release of the CTA's flag
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tid == 64) {
                K5S(l, 5);
                const int v = 16 * epoch + l + 1;
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(v) : "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAccCols) : "memory");
}

// Layer 17 on the tensor cores: out = x - conv(h, w17).  The single output channel is padded to
// N = 16 (the smallest UMMA N at M = 128), so a 128-px row segment is 36 UMMAs M=128 x N=16 x K=16
// (9 taps x 4 K-steps) into a 16-column fp32 accumulator; the epilogue reads column 0 only and writes
// the fp32 residual.  Same warp roles, halo ring and TMA map as k_conv64_tc (one row per unit);
// weights [9 taps][8 ic-groups][16 oc][8 ic] bf16 (18 KB, oc 1..15 zero).
constexpr int kLOC = 16;
constexpr int kLWBytes = 9 * 8 * kLOC * 16;  // 18,432
constexpr uint32_t kIdescL = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLOC >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
constexpr int kLSmem = kLWBytes + kSlots * kSlotBytes + 1024;

__global__ void __launch_bounds__(192, 1) k_conv_last_tc(const __grid_constant__ CUtensorMap amap,
                                                         const __nv_bfloat16* __restrict__ wts,
                                                         const float* __restrict__ x, float* out, int H, int W,
                                                         int rows_per_cta)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;
    unsigned char* slots = sm + kLWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;
    uint64_t* sfull = bars + 1;
    uint64_t* sempty = sfull + kSlots;
    uint64_t* afull = sempty + kSlots;
    uint64_t* aempty = afull + kAcc;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kAcc);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips;
    const int x0 = strip * kTileX;
    const int y0 = (blockIdx.x / strips) * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    if (y0 >= H) return;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kAcc * kLOC)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(sempty + i, 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            mbar_init(afull + i, 1);
            mbar_init(aempty + i, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;
    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            mbar_expect(wbar, kLWBytes);
            bulk_copy(sw, wts, kLWBytes, wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the last 64-channel layer
            for (int r = y0 - 1; r <= y1; ++r) {
                const int q = r - rbase, s = q % kSlots, u = q / kSlots;
                if (u >= 1) mbar_wait(sempty + s, (uint32_t)((u - 1) & 1));
                mbar_expect(sfull + s, kSlotBytes);
                tma_row(slots + s * kSlotBytes, &amap, x0 / 8 - 1, r, sfull + s);
            }
        }
    } else if (warp == 1) {  // ---- MMA issuer (whole warp, one elected lane issues)
        const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
        mbar_wait(wbar, 0);
        for (int y = y0; y < y1; ++y) {
            const int t = y - y0, b = t % kAcc, ub = t / kAcc;
            if (ub >= 1) mbar_wait(aempty + b, (uint32_t)((ub - 1) & 1));
            for (int r = y - 1; r <= y + 1; ++r) {
                const int q = r - rbase;
                mbar_wait(sfull + q % kSlots, (uint32_t)((q / kSlots) & 1));
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tmem + (uint32_t)(b * kLOC);
            const uint64_t b0 = sdesc(sw_base, kLOC * 16, 128);
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
                const uint64_t a0 = sdesc(sl_base + ((y - 1 + dy - rbase) % kSlots) * kSlotBytes, kHaloX * 16, 128);
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t a = a0 + (uint64_t)(((kHaloOff + dx) * 16 + 2 * j * (kHaloX * 16)) >> 4);
                        const uint64_t bd = b0 + (uint64_t)(((dy * 3 + dx) * (8 * kLOC * 16) + 2 * j * (kLOC * 16)) >> 4);
                        umma_e(d, a, bd, kIdescL, (dy | dx | j) != 0);
                    }
                }
            }
            umma_commit_e(afull + b);
            umma_commit_e(sempty + (y - 1 - rbase) % kSlots);  // row y-1: last reader was row y
        }
    } else {  // ---- epilogue warps 2..5: column 0 of the accumulator -> out = x - net(x)
        const int quad = warp & 3;
        for (int y = y0; y < y1; ++y) {
            const int t = y - y0, b = t % kAcc, ub = t / kAcc;
            mbar_wait(afull + b, (uint32_t)(ub & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * kLOC);
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(base));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + b)) : "memory");
            const int px = x0 + quad * 32 + lane;
            if (px < W) {
                const size_t p = (size_t)y * W + px;
                out[p] = x[p] - __uint_as_float(v);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * kLOC) : "memory");
}

// Layer 17 with rolling accumulators (k_conv_last_roll, the default): k_conv_last_tc issues 36 N = 16 UMMAs
// per output row one by one and is bound by the issue path (~58 cycles each; 19.7 us per 512^2 layer under
// ncu against 17.7 us for a 64 -> 64 layer with 64 times the math).  Here, as in k_conv64_roll, every halo
// row is one run of UMMAs against [W_dy2 | W_dy1 | W_dy0] (16 padded output channels each, N = 48) into
// the 16-column accumulator slots of output rows r-1, r, r+1: 13 UMMAs per row instead of 36.
// Weights [dx 3][ic-group 8][dy2 | dy1 | dy0 x 16 oc][8 ic] bf16 (18 KB, oc 1..15 of each block zero).
constexpr uint32_t kIdescL32 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr uint32_t kIdescL48 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(48 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr int kLRIcg = 3 * kLOC * 16;  // 768 B per ic-group: 48 output-channel rows of 8 ic
constexpr int kLRDx = 8 * kLRIcg;      // 6,144 B per dx
// (A, B) descriptor steps of the 11 (dx, K-step) UMMAs after the first: A as in umma_row12, B dx x 6,144 + 2 j x 768 (>> 4)
#define K5_STEPS_LAST(X) X(288, 96) X(576, 192) X(864, 288) X(1, 384) X(289, 480) X(577, 576) X(865, 672) X(2, 768) \
    X(290, 864) X(578, 960) X(866, 1056)
#define K5_STEP3(ao, bo) "add.s64 a, %1, " #ao ";\nadd.s64 b, %2, " #bo ";\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
#define K5_STEP5(ao, bo) "add.s64 a, %1, " #ao ";\nadd.s64 b, %2, " #bo ";\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n"
__device__ __forceinline__ void umma_last12(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t accumulate)
{
    static_assert(kHaloX == 144 && kLRDx == 6144 && kLRIcg == 768, "offsets are hard-coded");
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 1, 1;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        K5_STEPS_LAST(K5_STEP3)
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_last11(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc)
{
    asm volatile(
        "{\n.reg .pred e, t;\n.reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.eq.b32 t, 1, 1;\n"
        K5_STEPS_LAST(K5_STEP3)
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void umma_last13(uint32_t d_tmem, uint64_t a0, uint64_t b0)
{
    asm volatile(
        "{\n.reg .pred e, f, t;\n.reg .b64 a, b;\n.reg .b32 d2;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.eq.b32 t, 1, 1;\nsetp.ne.b32 f, 1, 1;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, t;\n"  // rows r-1, r: += A [W_dy2 | W_dy1]
        "add.u32 d2, %0, 32;\nadd.s64 b, %2, 32;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [d2], %1, b, %4, f;\n"   // row r+1: = A W_dy0
        K5_STEPS_LAST(K5_STEP5)
        "}\n"
        ::"r"(d_tmem), "l"(a0), "l"(b0), "r"(kIdescL32), "r"(kIdescL), "r"(kIdescL48)
        : "memory");
}
#undef K5_STEP3
#undef K5_STEP5

__global__ void __launch_bounds__(192, 1) k_conv_last_roll(const __grid_constant__ CUtensorMap amap,
                                                           const __nv_bfloat16* __restrict__ wts,
                                                           const float* __restrict__ x, float* out, int H, int W,
                                                           int rows_per_cta)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sw = sm;
    unsigned char* slots = sm + kLWBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kSlots * kSlotBytes);
    uint64_t* wbar = bars;
    uint64_t* sfull = bars + 1;             // [kSlots] halo row landed
    uint64_t* rowdone = sfull + kSlots;     // [kSlots] the halo row's UMMAs have completed
    uint64_t* aempty = rowdone + kSlots;    // [kRollAcc] accumulator slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kRollAcc);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int strips = (W + kTileX - 1) / kTileX;
    const int strip = blockIdx.x % strips;
    const int x0 = strip * kTileX;
    const int y0 = (blockIdx.x / strips) * rows_per_cta;
    const int y1 = min(H, y0 + rows_per_cta);
    if (y0 >= H) return;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                     "n"(kRollAcc * kLOC)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(wbar, 1);
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(sfull + i, 1);
            mbar_init(rowdone + i, 1);
        }
        for (int i = 0; i < kRollAcc; ++i) mbar_init(aempty + i, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int rbase = y0 - 1;
    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            mbar_expect(wbar, kLWBytes);
            bulk_copy(sw, wts, kLWBytes, wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the last 64-channel layer
            for (int r = y0 - 1; r <= y1; ++r) {
                const int q = r - rbase, s = q % kSlots, u = q / kSlots;
                if (u >= 1) mbar_wait(rowdone + s, (uint32_t)((u - 1) & 1));
                mbar_expect(sfull + s, kSlotBytes);
                tma_row(slots + s * kSlotBytes, &amap, x0 / 8 - 1, r, sfull + s);
            }
        }
    } else if (warp == 1) {  // ---- MMA issuer (whole warp, one elected lane issues)
        const uint32_t sw_base = s_u32(sw), sl_base = s_u32(slots);
        mbar_wait(wbar, 0);
        for (int r = y0 - 1; r <= y1; ++r) {
            const int q = r - rbase, s = q % kSlots;
            const bool v0 = r - 1 >= y0, v1 = r >= y0 && r < y1, v2 = r + 1 < y1;
            if (v2 && q >= kRollAcc) mbar_wait(aempty + (q % kRollAcc), (uint32_t)((q / kRollAcc - 1) & 1));
            mbar_wait(sfull + s, (uint32_t)((q / kSlots) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t a0 = sdesc(sl_base + s * kSlotBytes + kHaloOff * 16, kHaloX * 16, 128);
            const int s0 = (q + 2 * kRollAcc - 2) % kRollAcc;  // slot of output row r-1
            auto bd = [&](int k) { return sdesc(sw_base + k * kLOC * 16, kLRIcg, 128); };
            auto dc = [&](int k) { return tmem + (uint32_t)(((s0 + k) % kRollAcc) * kLOC); };
            if (v0 && v1 && v2 && s0 + 2 < kRollAcc) {
                umma_last13(dc(0), a0, bd(0));
            } else if (v0 && v1 && v2 && s0 + 1 < kRollAcc) {  // slots 6, 7 | 0
                umma_last12(dc(0), a0, bd(0), kIdescL32, 1u);
                umma_last12(dc(2), a0, bd(2), kIdescL, 0u);
            } else if (v0 && v1 && !v2 && s0 + 1 < kRollAcc) {  // the CTA's last image row
                umma_last12(dc(0), a0, bd(0), kIdescL32, 1u);
            } else {  // first rows, top and bottom halo rows, short CTAs, the other wrapping row
                if (v0) umma_last12(dc(0), a0, bd(0), kIdescL, 1u);
                if (v1) umma_last12(dc(1), a0, bd(1), kIdescL, 1u);
                if (v2) umma_last12(dc(2), a0, bd(2), kIdescL, 0u);
            }
            umma_commit_e(rowdone + s);
        }
    } else {  // ---- epilogue warps 2..5: column 0 of the row's accumulator slot -> out = x - net(x)
        const int quad = warp & 3;
        for (int y = y0; y < y1; ++y) {
            const int q = y + 1 - rbase, a = (y - y0) % kRollAcc;
            mbar_wait(rowdone + q % kSlots, (uint32_t)((q / kSlots) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * kLOC);
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(base));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(aempty + a)) : "memory");
            const int px = x0 + quad * 32 + lane;
            if (px < W) {
                const size_t p = (size_t)y * W + px;
                out[p] = x[p] - __uint_as_float(v);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kRollAcc * kLOC) : "memory");
}

// layer 1: x (fp32, rounded to bf16) -> 64 ch, ReLU, bf16 blocked [8][H][W][8].  w1: [9 taps][64 oc] fp32
// packed fp32 FMA (sm_100 FFMA2): {a.x * b.x + c.x, a.y * b.y + c.y}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c)
{
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}

__global__ void k_conv_first(const float* __restrict__ x, const __grid_constant__ ConvW9 w1, __nv_bfloat16* out,
                             int H, int W, int Wp)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= H * W) return;
    const int yy = p / W, xx = p % W;
    float in[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int sy = yy + t / 3 - 1, sx = xx + t % 3 - 1;
        in[t] = (sy >= 0 && sy < H && sx >= 0 && sx < W) ? __bfloat162float(__float2bfloat16_rn(x[sy * W + sx])) : 0.f;
    }
    uint4* dst = reinterpret_cast<uint4*>(out) + ((size_t)yy * Wp + xx);  // channel-blocked [group][H][Wp][8]
    const size_t gstride = (size_t)H * Wp;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t pk[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            // output channels oc, oc + 1 as one packed pair (FFMA2): same products and order as two FMAs
            const int oc = 8 * q + 2 * h;
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int t = 0; t < 9; ++t)
                acc = ffma2(make_float2(in[t], in[t]), make_float2(w1.v[t * kC + oc], w1.v[t * kC + oc + 1]), acc);
            const __nv_bfloat162 v2 = __floats2bfloat162_rn(fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f));
            pk[h] = *reinterpret_cast<const uint32_t*>(&v2);
        }
        dst[q * gstride] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// layer 17 + residual: out = x - sum_taps sum_ic h[ic] w17[tap][ic]  (fp32).  16 x 16 output pixels
// per block; the 18 x 18 x 64-channel input tile is staged once in shared memory (coalesced 16-byte
// loads, zero outside the image), then every pixel reads its 9 taps from there.
constexpr int kLastT = 16;
__global__ void __launch_bounds__(kLastT * kLastT) k_conv_last(const __nv_bfloat16* __restrict__ h,
                                                                const __grid_constant__ ConvW9 w17,
                                                                const float* __restrict__ x, float* out, int H, int W,
                                                                int Wp)
{
    constexpr int TT = kLastT + 2;
    __shared__ uint4 tile[4][TT][TT];  // four channel groups at a time: 20.7 KB, so a wave holds the grid
    const int tid = threadIdx.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the last 64-channel layer
    const int bx = blockIdx.x * kLastT, by = blockIdx.y * kLastT;
    const size_t gstride = (size_t)H * Wp;
    const int tx = tid % kLastT, ty = tid / kLastT;
    const int xx = bx + tx, yy = by + ty;
    float2 acc2 = make_float2(0.f, 0.f);  // even / odd channels
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        if (half) __syncthreads();  // every read of the first half is done
        for (int i = tid; i < 4 * TT * TT; i += blockDim.x) {
            const int g = i / (TT * TT), r = (i / TT) % TT, c = i % TT;
            const int sy = by + r - 1, sx = bx + c - 1;
            tile[g][r][c] = (sy >= 0 && sy < H && sx >= 0 && sx < W)
                                ? __ldg(reinterpret_cast<const uint4*>(h) + (4 * half + g) * gstride + (size_t)sy * Wp + sx)
                                : make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 9; ++t) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = tile[q][ty + t / 3][tx + t % 3];
                const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {  // bf16 pair -> fp32 pair by shifts, one FFMA2 per pair
                    const float2 f = make_float2(__uint_as_float(u[e] << 16), __uint_as_float(u[e] & 0xffff0000u));
                    const int c = t * kC + 8 * (4 * half + q) + 2 * e;
                    acc2 = ffma2(f, make_float2(w17.v[c], w17.v[c + 1]), acc2);
                }
            }
        }
    }
    if (xx >= W || yy >= H) return;
    const size_t p = (size_t)yy * W + xx;
    out[p] = x[p] - (acc2.x + acc2.y);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 4-D view of a channel-blocked [8][H][Wp][8] bf16 image (row pitch Wp = W rounded up to 8 px,
// padding columns zero) in 8-pixel chunks: (64 elements = 8 px x 8 ch, x chunk, y, group 8),
// box {64, 18, 1, 8}: every TMA row is 128 B
CUtensorMap make_act_map(void* base, int H, int Wp)
{
    CUtensorMap m;
    const cuuint64_t dims[4] = {64, (cuuint64_t)Wp / 8, (cuuint64_t)H, 8};
    // a halo row of one group is 144 x 16 B contiguous
    const cuuint64_t strides[3] = {128, (cuuint64_t)Wp * 16, (cuuint64_t)H * Wp * 16};  // bytes, dims 1..3
    const cuuint32_t box[4] = {64, (cuuint32_t)(kHaloX / 8), 1, 8};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

#define CKC(x)                                                                                             \
    do {                                                                                                   \
        cudaError_t e_ = (x);                                                                              \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#ifdef K5_TRACE
void k5_trace_copy(long long* host) { cudaMemcpyFromSymbol(host, g_k5_trace, sizeof(g_k5_trace)); }
unsigned k5_life_copy(long long* host, bool reset)
{
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, g_k5_life_n, sizeof(n));
    cudaMemcpyFromSymbol(host, g_k5_life, sizeof(g_k5_life));
    if (reset) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(g_k5_life_n, &z, sizeof(z));
    }
    return n;
}
#endif
#ifdef K5SEQ_TRACE
extern "C" int mace_k5seq_trace(unsigned long long* host)
{
    return cudaMemcpyFromSymbol(host, g_k5seq, sizeof(g_k5seq)) == cudaSuccess ? 0 : -1;
}
#endif

void Cnn::set_weights(const uint16_t* bf16, int layers, int channels)
{
    if (layers != 17 || channels != kC) throw std::runtime_error("the denoiser is 17 layers x 64 channels");
    // input layout per layer l: PyTorch OIHW [oc][ic][3][3] as bf16 bits
    const size_t n1 = (size_t)kC * 1 * 9, nm = (size_t)kC * kC * 9, n17 = (size_t)1 * kC * 9;
    auto f = [](uint16_t b) {
        uint32_t u = (uint32_t)b << 16;
        float v;
        std::memcpy(&v, &u, 4);
        return v;
    };
    for (int oc = 0; oc < kC; ++oc)
        for (int t = 0; t < 9; ++t) w_first.v[t * kC + oc] = f(bf16[oc * 9 + t]);
    const uint16_t* wl = bf16 + n1 + 15 * nm;
    for (int ic = 0; ic < kC; ++ic)
        for (int t = 0; t < 9; ++t) w_last.v[t * kC + ic] = f(wl[ic * 9 + t]);
    // layer 17 for the tensor cores: [tap][ic-group][16 oc][8 ic], output channel 0 only
    {
        std::vector<uint16_t> wt((size_t)kLWBytes / 2, 0);
        for (int ic = 0; ic < kC; ++ic)
            for (int t = 0; t < 9; ++t) wt[(size_t)t * 8 * kLOC * 8 + (ic / 8) * kLOC * 8 + ic % 8] = wl[ic * 9 + t];
        w_last_tc.alloc(wt.size());
        CKC(cudaMemcpy(w_last_tc.p, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice));
    }
    // ... and for k_conv_last_roll: [dx][ic-group][dy2 | dy1 | dy0 x 16 oc][8 ic], output channel 0 of each block
    {
        std::vector<uint16_t> wt((size_t)kLWBytes / 2, 0);
        for (int ic = 0; ic < kC; ++ic)
            for (int dy = 0; dy < 3; ++dy)
                for (int dx = 0; dx < 3; ++dx)
                    wt[(size_t)dx * kLRDx / 2 + (ic / 8) * kLRIcg / 2 + (2 - dy) * kLOC * 8 + ic % 8] = wl[ic * 9 + dy * 3 + dx];
        w_last_roll.alloc(wt.size());
        CKC(cudaMemcpy(w_last_roll.p, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice));
    }
    const char* el = std::getenv("MACE_K5_LAST");  // "fma": layer 17 on the CUDA cores; "tc": one UMMA run per output row
    last_tc = !(el && std::strcmp(el, "fma") == 0);
    last_roll = !(el && (std::strcmp(el, "fma") == 0 || std::strcmp(el, "tc") == 0));
    const char* es = std::getenv("MACE_K5_SEQ");  // "1": the 15 middle layers as one persistent launch
    seq = es && std::strcmp(es, "1") == 0;
    seq_pipe = es && std::strcmp(es, "2") == 0;  // "2": pipelined persistent launch (k_conv64_pipe)
    // middle layers: [layer][tap][ic-group][oc][8 ic]
    std::vector<uint16_t> wm(15 * (size_t)9 * kC * kC);
    for (int l = 0; l < 15; ++l) {
        const uint16_t* src = bf16 + n1 + l * nm;
        uint16_t* dst = wm.data() + (size_t)l * 9 * kC * kC;
        for (int oc = 0; oc < kC; ++oc)
            for (int ic = 0; ic < kC; ++ic)
                for (int t = 0; t < 9; ++t)
                    dst[(size_t)t * kC * kC + (ic / 8) * kC * 8 + oc * 8 + (ic % 8)] = src[(oc * kC + ic) * 9 + t];
    }
    // row-pair layout: for each dx and ic-group, the three dy taps' [64 oc][8 ic] blocks side by side
    // in the order dy2, dy1, dy0 (k_conv64_tc2)
    std::vector<uint16_t> wm2(wm.size());
    for (int l = 0; l < 15; ++l) {
        const uint16_t* src = bf16 + n1 + l * nm;
        uint16_t* dst = wm2.data() + (size_t)l * 9 * kC * kC;
        for (int oc = 0; oc < kC; ++oc)
            for (int ic = 0; ic < kC; ++ic)
                for (int dy = 0; dy < 3; ++dy)
                    for (int dx = 0; dx < 3; ++dx)
                        dst[(size_t)dx * kW2Dx / 2 + (ic / 8) * kW2Icg / 2 + (2 - dy) * kC * 8 + oc * 8 + (ic % 8)] =
                            src[(oc * kC + ic) * 9 + dy * 3 + dx];
    }
    w_mid2.alloc(wm2.size());
    CKC(cudaMemcpy(w_mid2.p, wm2.data(), wm2.size() * 2, cudaMemcpyHostToDevice));
    const char* ev = std::getenv("MACE_K5_ROWS");  // output rows per MMA unit: 1, 2 or 3; 0 = rolling accumulators
    rows_unit = ev ? std::max(0, std::min(3, std::atoi(ev))) : 0;
    (void)n17;

    w_mid.alloc(wm.size());

    CKC(cudaMemcpy(w_mid.p, wm.data(), wm.size() * 2, cudaMemcpyHostToDevice));
    ready = true;
}

void Cnn::ensure(int h, int w)
{
    if (h == H && w == W && act0.p) return;
    H = h;
    W = w;
    Wp = (w + 7) & ~7;
    act0.alloc((size_t)H * Wp * kC);
    act1.alloc((size_t)H * Wp * kC);
    CKC(cudaMemset(act0.p, 0, (size_t)H * Wp * kC * 2));  // padding columns stay zero (never written)
    CKC(cudaMemset(act1.p, 0, (size_t)H * Wp * kC * 2));
    map0 = make_act_map(act0.p, H, Wp);
    map1 = make_act_map(act1.p, H, Wp);
    CKC(cudaFuncSetAttribute(k_conv64_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    CKC(cudaFuncSetAttribute(k_conv64_tc2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    CKC(cudaFuncSetAttribute(k_conv64_tc2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    CKC(cudaFuncSetAttribute(k_conv64_roll<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    CKC(cudaFuncSetAttribute(k_conv64_roll<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    CKC(cudaFuncSetAttribute(k_conv64_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
    CKC(cudaFuncSetAttribute(k_conv_last_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kLSmem));
    CKC(cudaFuncSetAttribute(k_conv_last_roll, cudaFuncAttributeMaxDynamicSharedMemorySize, kLSmem));
    CKC(cudaFuncSetAttribute(k_conv64_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    flags.alloc(1024);
    CKC(cudaMemset(flags.p, 0, 1024 * sizeof(int)));
    epoch = 0;
    roll_epoch = 0;
    pflags.alloc(4096);
    CKC(cudaMemset(pflags.p, 0, 4096 * sizeof(int)));
    pipe_epoch = 0;
}

// one 64 -> 64 layer (2..16) from map -> dst on stream s with the current launch geometry
void Cnn::launch_mid(int l, const CUtensorMap& m, __nv_bfloat16* dst, cudaStream_t s, int num_sms, bool pdl_on)
{
    // one CTA per (128-px strip, run of rows); one CTA per SM (140 KB smem)
    const int strips = (W + kTileX - 1) / kTileX;
    const int ctas_y = std::max(1, num_sms / strips);
    const int per = (H + ctas_y - 1) / ctas_y;  // rows per CTA
    const int ctas = strips * ((H + per - 1) / per);
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = pdl_on ? 1 : 0;
    if (rows_unit == 0)
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_roll<false>, m, m, (const __nv_bfloat16*)(w_mid2.p + (size_t)l * 9 * kC * kC),
                               dst, dst, H, W, Wp, per, 1, (unsigned*)nullptr, 0u));
    else if (rows_unit == 3)
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_tc2<3>, m, (const __nv_bfloat16*)(w_mid2.p + (size_t)l * 9 * kC * kC),
                               dst, H, W, Wp, per));
    else if (rows_unit == 2)
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_tc2<2>, m, (const __nv_bfloat16*)(w_mid2.p + (size_t)l * 9 * kC * kC),
                               dst, H, W, Wp, per));
    else
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_tc, m, (const __nv_bfloat16*)(w_mid.p + (size_t)l * 9 * kC * kC), dst,
                               H, W, Wp, per));
}

void Cnn::layer(int l, const uint16_t* in_chw, uint16_t* out_chw, int h, int w, cudaStream_t s, int num_sms)
{
    if (!ready) throw std::runtime_error("denoiser weights not set");
    if (l < 0 || l >= 15) throw std::runtime_error("middle layer index 0..14");
    ensure(h, w);
    // CHW bf16 -> channel-blocked [8 groups][H][Wp][8 ch] (padding columns zero)
    std::vector<uint16_t> blk((size_t)H * Wp * kC, 0);
    for (int c = 0; c < kC; ++c)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                blk[(((size_t)(c / 8) * H + y) * Wp + x) * 8 + (c % 8)] = in_chw[((size_t)c * H + y) * W + x];
    CKC(cudaMemcpyAsync(act0.p, blk.data(), blk.size() * 2, cudaMemcpyHostToDevice, s));
    launch_mid(l, map0, act1.p, s, num_sms, false);
    CKC(cudaMemcpyAsync(blk.data(), act1.p, blk.size() * 2, cudaMemcpyDeviceToHost, s));
    CKC(cudaStreamSynchronize(s));
    for (int c = 0; c < kC; ++c)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                out_chw[((size_t)c * H + y) * W + x] = blk[(((size_t)(c / 8) * H + y) * Wp + x) * 8 + (c % 8)];
}

void Cnn::apply(const float* x, float* out, int h, int w, cudaStream_t s, int num_sms, int* launches)
{
    if (!ready) throw std::runtime_error("denoiser weights not set");
    ensure(h, w);
    const int npx = H * W;
    k_conv_first<<<(npx + 255) / 256, 256, 0, s>>>(x, w_first, act0.p, H, W, Wp);
    // layers 2..17 are launched with programmatic stream serialization (PDL): each one's prologue
    // overlaps the previous layer's tail; griddepcontrol.wait orders the activation reads
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    if (seq_pipe && rows_unit == 0) {  // rolling accumulators, pipelined layers (half-run shifts, row flags)
        const int strips = (W + kTileX - 1) / kTileX;
        const int ctas_y = std::max(1, num_sms / strips);
        const int per = (H + ctas_y - 1) / ctas_y;
        const int nyc = (H + per - 1) / per;
        const int ctas = strips * nyc;
        if (ctas * 8 > 4096) throw std::runtime_error("denoiser grid too large");
        cudaLaunchAttribute coop[1];
        coop[0].id = cudaLaunchAttributeCooperative;
        coop[0].val.cooperative = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(kPThreads);
        cfg.dynamicSmemBytes = kPSmem;
        cfg.stream = s;
        cfg.attrs = coop;
        cfg.numAttrs = 1;
        // flag values run on from denoise to denoise: a run publishes at most 15 x (rows per run + per / 2) < 2^16
        const unsigned base = (unsigned)pipe_epoch << 16;
        ++pipe_epoch;
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_pipe, map0, map1, (const __nv_bfloat16*)w_mid2.p, act1.p, act0.p, H, W, Wp,
                               per, 15, (unsigned*)pflags.p, base));
    } else if (seq && rows_unit == 0) {  // rolling accumulators, the 15 middle layers as one cooperative launch
        const int strips = (W + kTileX - 1) / kTileX;
        const int ctas_y = std::max(1, num_sms / strips);
        const int per = (H + ctas_y - 1) / ctas_y;
        const int ctas = strips * ((H + per - 1) / per);
        cudaLaunchAttribute coop[1];
        coop[0].id = cudaLaunchAttributeCooperative;
        coop[0].val.cooperative = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = s;
        cfg.attrs = coop;
        cfg.numAttrs = 1;
        // arrivals so far on the grid-wide counter (flags[1023]): 14 per CTA and denoise at this geometry
        const unsigned base = (unsigned)roll_epoch * 14u * (unsigned)ctas;
        ++roll_epoch;
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_roll<true>, map0, map1, (const __nv_bfloat16*)w_mid2.p, act1.p, act0.p, H,
                               W, Wp, per, 15, (unsigned*)(flags.p + 1023), base));
    } else if (seq && rows_unit == 2) {  // the 15 middle layers as one persistent cooperative launch
        const int strips = (W + kTileX - 1) / kTileX;
        const int ctas_y = std::max(1, num_sms / strips);
        const int per = (H + ctas_y - 1) / ctas_y;
        const int ctas = strips * ((H + per - 1) / per);
        if (ctas > 1024) throw std::runtime_error("denoiser grid too large");
        ++epoch;
        cudaLaunchAttribute coop[1];
        coop[0].id = cudaLaunchAttributeCooperative;
        coop[0].val.cooperative = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = s;
        cfg.attrs = coop;
        cfg.numAttrs = 1;
        CKC(cudaLaunchKernelEx(&cfg, k_conv64_seq, map0, map1, (const __nv_bfloat16*)w_mid2.p, act0.p, act1.p, H, W,
                               Wp, per, 15, flags.p, epoch));
    } else {
        for (int l = 0; l < 15; ++l)
            launch_mid(l, (l & 1) ? map1 : map0, (l & 1) ? act0.p : act1.p, s, num_sms, true);
    }
    // 15 middle layers: the last one wrote act1 (l = 14 even -> dst act1)
    if (last_tc) {
        const int strips = (W + kTileX - 1) / kTileX;
        const int ctas_y = std::max(1, num_sms / strips);
        const int per = (H + ctas_y - 1) / ctas_y;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(strips * ((H + per - 1) / per));
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = kLSmem;
        cfg.stream = s;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        if (last_roll)
            CKC(cudaLaunchKernelEx(&cfg, k_conv_last_roll, map1, (const __nv_bfloat16*)w_last_roll.p, x, out, H, W, per));
        else
            CKC(cudaLaunchKernelEx(&cfg, k_conv_last_tc, map1, (const __nv_bfloat16*)w_last_tc.p, x, out, H, W, per));
    } else {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((W + kLastT - 1) / kLastT, (H + kLastT - 1) / kLastT);
        cfg.blockDim = dim3(kLastT * kLastT);
        cfg.stream = s;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        CKC(cudaLaunchKernelEx(&cfg, k_conv_last, (const __nv_bfloat16*)act1.p, w_last, x, out, H, W,
                               Wp));
    }
    CKC(cudaGetLastError());
    if (launches) *launches += 17;
}

}  // namespace mace
