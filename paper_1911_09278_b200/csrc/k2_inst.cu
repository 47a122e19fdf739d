// K2 super-voxel launch for one tile side (compiled once per S with -DMACE_SV_SIDE=S by
// _build.py): the k_icd_sv<S, K, NG, weighted> instantiations and their occupancy-bounded grid.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "k2_launch.h"
#include "k_sv.cuh"

#ifndef MACE_SV_SIDE
#error "compile k2_inst.cu with -DMACE_SV_SIDE=<tile side>"
#endif

namespace mace {
namespace {

void ck(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <int S, int K, int NG, bool kW, int MW = 0>
void launch(SvLaunch& L, const PassParams& P)
{
    auto kern = k_icd_sv<S, K, NG, kW, MW>;
    const int wpb = MW ? L.chunks : kSvThreads / 32;  // warps per block (one tile per block when MW)
    // occupancy of this instantiation at this shared-memory size, queried once per (device, size);
    // the kernel's dynamic shared-memory limit only ever grows (per device)
    static thread_local std::vector<std::pair<std::pair<int, size_t>, int>> occ;
    static thread_local std::vector<std::pair<int, size_t>> limit;
    size_t* lim = nullptr;
    for (auto& e : limit)
        if (e.first == L.device) lim = &e.second;
    if (!lim) {
        limit.push_back({L.device, 0});
        lim = &limit.back().second;
    }
    if (L.smem > *lim) {
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem), "K2 smem attribute");
        *lim = L.smem;
    }
    int nb = -1;
    for (auto& e : occ)
        if (e.first.first == L.device && e.first.second == L.smem) nb = e.second;
    if (nb < 0) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * wpb, L.smem), "K2 occupancy");
        occ.push_back({{L.device, L.smem}, nb});
    }
    if (nb < 1) throw std::runtime_error("super-voxel kernel does not fit on an SM (band too large)");
    // Concurrency bound: at most a fraction `frac` of the queue's tiles are in flight at once
    // (bounded staleness), never fewer than one tile per agent, never more than
    // the resident warps of the whole GPU.
    if (MW) {  // one tile per block: the bound is on blocks
        long blocks = (long)nb * L.num_sms;
        long cap = (long)std::floor(L.frac * (double)P.n_items);
        cap = std::max<long>(cap, L.agents_in_queue);
        if (L.max_warps > 0) cap = std::min<long>(cap, std::max(1L, L.max_warps / wpb));
        blocks = std::max(1L, std::min(blocks, cap));
        L.grid = (int)blocks;
        L.warps = (int)(blocks * wpb);
        kern<<<(int)blocks, 32 * wpb, L.smem, L.stream>>>(P);
        ck(cudaGetLastError(), "K2 launch");
        return;
    }
    long warps = (long)nb * wpb * L.num_sms;
    long cap = (long)std::floor(L.frac * (double)P.n_items);
    cap = std::max<long>(cap, L.agents_in_queue);
    if (L.max_warps > 0) cap = std::min<long>(cap, L.max_warps);
    warps = std::max(1L, std::min(warps, cap));
    const int threads = warps >= wpb ? kSvThreads : (int)warps * 32;
    const long grid = warps >= wpb ? warps / wpb : 1;
    L.grid = (int)grid;
    L.warps = (int)(grid * threads / 32);
    kern<<<(int)grid, threads, L.smem, L.stream>>>(P);
    ck(cudaGetLastError(), "K2 launch");
}

template <int K, int NG>
void by_weight(SvLaunch& L, const PassParams& P)
{
    if (L.weighted) launch<MACE_SV_SIDE, K, NG, true>(L, P);
    else launch<MACE_SV_SIDE, K, NG, false>(L, P);
}

template <int K>
void by_groups(SvLaunch& L, const PassParams& P)
{
    if (L.chunks > 1) {  // multi-warp tiles: 3 groups per chunk, K = 2 (layout.cpp)
        if constexpr (K == 2) {
            if (L.NG != 3) throw std::runtime_error("multi-warp tiles need 3 view groups per chunk");
            if (L.chunks > kSvMaxChunksDev) throw std::runtime_error("too many view chunks per tile");
            if (L.chunks <= 8) {
                if (L.weighted) launch<MACE_SV_SIDE, 2, 3, true, 1>(L, P);
                else launch<MACE_SV_SIDE, 2, 3, false, 1>(L, P);
            } else {
                if (L.weighted) launch<MACE_SV_SIDE, 2, 3, true, 2>(L, P);
                else launch<MACE_SV_SIDE, 2, 3, false, 2>(L, P);
            }
            return;
        } else {
            throw std::runtime_error("multi-warp tiles need K = 2");
        }
    }
    switch (L.NG) {
        case 1: by_weight<K, 1>(L, P); break;
        case 2: by_weight<K, 2>(L, P); break;
        case 3: by_weight<K, 3>(L, P); break;
        default: by_weight<K, 4>(L, P); break;
    }
}

}  // namespace

#define MACE_CAT2(a, b) a##b
#define MACE_CAT(a, b) MACE_CAT2(a, b)
void MACE_CAT(sv_launch_s, MACE_SV_SIDE)(SvLaunch& L, const PassParams& P)
{
    if (L.K <= 2) by_groups<2>(L, P);
    else by_groups<4>(L, P);
}

}  // namespace mace
