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

template <int S, int K, int NG, bool kW>
void launch(SvLaunch& L, const PassParams& P)
{
    auto kern = k_icd_sv<S, K, NG, kW>;
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
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kSvThreads, L.smem), "K2 occupancy");
        occ.push_back({{L.device, L.smem}, nb});
    }
    if (nb < 1) throw std::runtime_error("super-voxel kernel does not fit on an SM (band too large)");
    // Concurrency bound: at most a fraction `frac` of the queue's tiles are in flight at once
    // (bounded staleness), never fewer than one tile per agent, never more than
    // the resident warps of the whole GPU.
    constexpr int wpb = kSvThreads / 32;
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
