// Host interface of the super-voxel K2 launch (k_sv.cuh), compiled once per tile side S in
// k2_inst.cu (-DMACE_SV_SIDE=S), so the instantiations build in parallel and mace.cu does not
// carry them.
#pragma once
#include <cuda_runtime.h>

#include "dev_common.cuh"

namespace mace {

constexpr int kSvThreads = 32;  // one warp per block: a block is one tile worker

// shared-memory bytes per warp: the band (per row unit u = g W + o: e, lambda and e0 as three
// 32-word lane vectors at word 96 u; weighted records: e and e0 at word 64 u), the state tile
// with halo, per-pixel v and w, and the batch's four {theta1, den, z, v} (64 B)
__host__ __device__ constexpr int sv_unit_words(bool weighted) { return weighted ? 64 : 96; }
__host__ __device__ constexpr size_t sv_warp_bytes(int S, int ng, int wcap, bool weighted)
{
    return 4 * (size_t)sv_unit_words(weighted) * ng * wcap + 4 * (size_t)((((S + 2) * (S + 2)) + 3) & ~3) +
           8 * (size_t)S * S + 64;
}

struct SvLaunch {
    int device = 0;
    cudaStream_t stream = nullptr;
    size_t smem = 0;               // dynamic shared memory per block
    int num_sms = 148;
    double frac = 1.0 / 16.0;      // max fraction of the queue's tiles in flight
    long max_warps = 0;            // optional hard cap (0: none)
    int agents_in_queue = 1;       // never fewer warps than this
    int K = 2, NG = 1;             // slot width and view groups of the records
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
