// Host interface of the super-voxel K2 launch (k_sv.cuh), compiled once per tile side S in
// k2_inst.cu (-DMACE_SV_SIDE=S), so the instantiations build in parallel and mace.cu does not
// carry them.
#pragma once
#include <cuda_runtime.h>

#include "dev_common.cuh"

namespace mace {

constexpr int kSvThreads = 32;  // one warp per block: a block is one tile worker
constexpr int kSvMaxChunksDev = 16;  // multi-warp tiles: warps per block (internal.h kSvMaxChunks)

#ifndef MACE_K2_RAW
// 1: the e windows are copied into a per-warp raw area by coalesced cp.async (four lanes per view,
// 8 views per instruction) and transposed into the banked band by the owning lane; the raw copy
// doubles as the snapshot e0 of the write-back (no e0 plane).  0: every lane loads its own view's
// window with 16-byte loads (32 lines per instruction) and stores e and e0 planes.
#define MACE_K2_RAW 0
#endif

// shared-memory bytes per warp: the band (per row unit u = g W + o: e and lambda as 32-word lane
// vectors at word 64 u; weighted records: e at word 32 u; without the raw area also an e0 plane),
// the state tile with halo, per-pixel v and w, the batch's four {theta1, den, z, v} (64 B), and
// [raw] the raw windows (per (group, lane) a slot of 4 q words, q odd so that the quarter-warps of
// a 16-byte read hit distinct bank quads)
__host__ __device__ constexpr int sv_unit_words(bool weighted)
{
    return MACE_K2_RAW ? (weighted ? 32 : 64) : (weighted ? 64 : 96);
}
__host__ __device__ constexpr int sv_raw_quads(int wcap) { return ((wcap + 6) >> 2) | 1; }
__host__ __device__ constexpr size_t sv_raw_bytes(int ng, int wcap)
{
    return MACE_K2_RAW ? 16 * (size_t)ng * 32 * sv_raw_quads(wcap) : 0;
}
__host__ __device__ constexpr size_t sv_warp_bytes(int S, int ng, int wcap, bool weighted)
{
    return 4 * (size_t)sv_unit_words(weighted) * ng * wcap + 4 * (size_t)((((S + 2) * (S + 2)) + 3) & ~3) +
           8 * (size_t)S * S + 64 + sv_raw_bytes(ng, wcap);
}

// multi-warp tiles: the block area after the warps' regions (k_sv.cuh): next-item slots, warp 0's
// tile-state snapshot (z with halo, w, v) and the theta1 partials [2][4][chunks]
__host__ __device__ constexpr size_t sv_block_extra_bytes(int S, int chunks)
{
    return chunks > 1 ? 16 + 4 * (size_t)((((S + 2) * (S + 2)) + 3) & ~3) + 8 * (size_t)S * S + 32 * (size_t)chunks : 0;
}

struct SvLaunch {
    int device = 0;
    cudaStream_t stream = nullptr;
    size_t smem = 0;               // dynamic shared memory per block
    int num_sms = 148;
    double frac = 1.0 / 16.0;      // max fraction of the queue's tiles in flight
    long max_warps = 0;            // optional hard cap (0: none)
    int agents_in_queue = 1;       // never fewer warps than this
    int K = 2, NG = 1;             // slot width and view groups of the records (per chunk)
    int chunks = 1;                // warps per tile (view chunks)
    bool weighted = false;         // records hold a sqrt(lambda): no lambda plane (k_sv.cuh)
    int grid = 0, warps = 0;       // out: the launch shape used
};

// Launch one K2 pass over P.queue[0, P.n_items) on L.stream (throws std::runtime_error).
void sv_launch_s2(SvLaunch& L, const PassParams& P);
void sv_launch_s4(SvLaunch& L, const PassParams& P);
void sv_launch_s6(SvLaunch& L, const PassParams& P);
void sv_launch_s8(SvLaunch& L, const PassParams& P);
void sv_launch_s12(SvLaunch& L, const PassParams& P);
void sv_launch_s16(SvLaunch& L, const PassParams& P);

}  // namespace mace
