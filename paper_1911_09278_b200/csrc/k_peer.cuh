// Consensus over NVLink peer memory: the consensus average (mace.py:71-90) and the stop-test
// norms (mace.py:309-318) across ranks, fused with the local tree sum, with no collective library
// on the data path.
//
// Every rank owns one symmetric buffer (allocated and exchanged by the host through
// torch.distributed's symmetric memory); all ranks can load and store every rank's buffer.
//   [flags: kMaxPeers x u32 epoch][norms: 2 parities x kMaxPeers x 8 f64][data: 2 parities x world x n f32]
// k_peer_push:   the local tree sum over this rank's agents (K4's tree, scale 1) is stored straight
//                into slot [parity][rank] of EVERY rank's buffer (remote stores over NVLink), plus the
//                5 local norm sums; the last block fences system-wide and raises flag[rank] = epoch in
//                every rank's buffer (st.release.sys).
// k_peer_reduce: waits for all ranks' flags in its own buffer (ld.acquire.sys), then sums the world
//                slots in rank order (deterministic, identical on every rank) -> wbar, sums5.
// Double buffering by iteration parity: a rank can run at most one iteration ahead of any peer (its
// next push needs this iteration's reduce everywhere), so slot [parity] is never overwritten while
// a slow peer still reads it.
#pragma once
#include "kernels.cuh"

namespace mace {

constexpr int kMaxPeers = 8;

struct PeerArgs {
    unsigned char* buf[kMaxPeers];  // every rank's symmetric buffer (buf[rank] = this rank's)
    int world, rank;
    int parity;
    uint32_t epoch;
};

__host__ __device__ constexpr size_t peer_norm_off() { return 256; }
__host__ __device__ constexpr size_t peer_data_off() { return 256 + 2 * kMaxPeers * 8 * 8; }
__host__ __device__ constexpr size_t peer_bytes(int world, size_t n) { return peer_data_off() + 2 * (size_t)world * n * 4; }

__device__ __forceinline__ float* peer_data(const PeerArgs& A, int owner, int parity, int src, size_t n)
{
    return reinterpret_cast<float*>(A.buf[owner] + peer_data_off()) + ((size_t)parity * A.world + src) * n;
}
__device__ __forceinline__ double* peer_norms(const PeerArgs& A, int owner, int parity, int src)
{
    return reinterpret_cast<double*>(A.buf[owner] + peer_norm_off()) + ((size_t)parity * kMaxPeers + src) * 8;
}

template <int NL>  // local agents (0: any, up to 64)
__global__ void k_peer_push(const float* W, int n_local, size_t n, const double* sums5, PeerArgs A,
                            unsigned* counter, const int* done)
{
    if (done && *done) return;  // identical on every rank: the reduced norms and the stop test are
    for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < n; s += (size_t)gridDim.x * blockDim.x) {
        float v;
        if constexpr (NL > 0) {
            float acc[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) acc[i] = __ldcg(W + (size_t)i * n + s);
            v = tree_sum<NL>(acc);
        } else {
            float acc[64];
            for (int i = 0; i < n_local; ++i) acc[i] = W[(size_t)i * n + s];
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
            v = acc[0];
        }
        for (int r = 0; r < A.world; ++r) __stcg(peer_data(A, r, A.parity, A.rank, n) + s, v);
    }
    if (blockIdx.x == 0 && threadIdx.x < 5)
        for (int r = 0; r < A.world; ++r) peer_norms(A, r, A.parity, A.rank)[threadIdx.x] = sums5[threadIdx.x];
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x < A.world) {
        __threadfence_system();
        uint32_t* flag = reinterpret_cast<uint32_t*>(A.buf[threadIdx.x]) + A.rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(A.epoch) : "memory");
        if (threadIdx.x == 0) *counter = 0u;
    }
}

__global__ void k_peer_reduce(PeerArgs A, size_t n, float scale, float* wbar, double* sums5, const int* done)
{
    if (done && *done) return;
    if (threadIdx.x < A.world) {
        const uint32_t* flag = reinterpret_cast<const uint32_t*>(A.buf[A.rank]) + threadIdx.x;
        uint32_t f = 0;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
        } while ((int32_t)(f - A.epoch) < 0);
    }
    __syncthreads();
    for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < n; s += (size_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int r = 0; r < A.world; ++r) acc += __ldcg(peer_data(A, A.rank, A.parity, r, n) + s);
        wbar[s] = acc / scale;
    }
    if (blockIdx.x == 0 && threadIdx.x < 5) {
        double acc = 0.0;
        for (int r = 0; r < A.world; ++r) acc += __ldcg(peer_norms(A, A.rank, A.parity, r) + threadIdx.x);
        sums5[threadIdx.x] = acc;
    }
}

}  // namespace mace
