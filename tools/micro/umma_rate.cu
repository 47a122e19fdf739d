// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16, SS operands, SWIZZLE_NONE)
// as a function of N, with A re-read every MMA vs kept in the A collector.  One CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

template <int N, int MODE>  // MODE 0 plain, 1 collector reuse (fill, use x k, lastuse)
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bars4[4];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tslot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
        for (int c = 0; c < 4; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bars4[c])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < (MODE >= 5 ? 200 : 48) * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x == 32) {
        const uint64_t a = sdesc(s_u32(sm), 130 * 16, 128);
        const uint64_t b = sdesc(s_u32(sm + 16384), N * 16, 128);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE == 0) {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
            } else if (MODE == 2 || MODE == 3) {  // distinct A tiles: 2 = 16-byte (1 px) shifted starts, 3 = aligned
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint64_t au = a + (uint64_t)(((MODE == 2 ? (u % 3) * 16 : 0) + (u / 3) * 256) >> 4);
                    const uint64_t bu = b + (uint64_t)((u * 256) >> 4);
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(au), "l"(bu), "r"(idesc));
                }
            } else if (MODE == 4) {  // K5 row-pair unit pattern: 2 x 12 N=128 then 2 x 12 N=64 (D at +0 / +64)
                constexpr uint32_t i128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t i64 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
#pragma unroll
                for (int u = 0; u < 48; ++u) {
                    const uint32_t id = u < 24 ? i128 : i64;
                    const uint32_t dd = tmem + (u >= 36 ? 64u : 0u);
                    const uint64_t au = a + (uint64_t)((((u % 3) * 16) + ((u / 3) % 4) * 256) >> 4);
                    const uint64_t bu = b + (uint64_t)(((u % 12) * 256) >> 4);
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dd), "l"(au), "l"(bu), "r"(id));
                }
            } else if (MODE >= 12 && MODE <= 15) {
                // one wrapping halo row of the rolling kernel: 12 x N=128 into columns 384.. and 12 x N=64 into
                // column 0.  12: the two runs one after the other; 13: interleaved; 14: as 12 with both runs in
                // adjacent columns (384 / 256); 15: regular row (N=128 + N=64 + 11 x N=192)
                constexpr uint32_t i192 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(192 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t i128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t i64 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                const uint32_t wb = s_u32(sm), sl = s_u32(sm) + 73728;
                const uint32_t dA = tmem + 384, dB = tmem + (MODE == 14 ? 256 : 0);
#pragma unroll
                for (int pass = 0; pass < (MODE == 13 || MODE == 15 ? 1 : 2); ++pass)
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint64_t au = sdesc(sl + (7 + dx) * 16 + 2 * j * 2304, 2304, 128);
                            const uint64_t bu = sdesc(wb + dx * 24576 + 2 * j * 3072, 3072, 128);
                            const uint64_t bu2 = sdesc(wb + 2048 + dx * 24576 + 2 * j * 3072, 3072, 128);
                            if (MODE == 15) {
                                if (dx == 0 && j == 0) {
                                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(au), "l"(bu), "r"(i128));
                                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 128), "l"(au), "l"(bu2), "r"(i64));
                                } else
                                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(au), "l"(bu), "r"(i192));
                            } else {
                                if (MODE == 13 || pass == 0)
                                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dA), "l"(au), "l"(bu), "r"(i128));
                                if (MODE == 13 || pass == 1)
                                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dB), "l"(au), "l"(bu2), "r"(i64));
                            }
                        }
            } else if (MODE >= 5 && MODE <= 11) {
                // K5 row-triple unit with the layer's own descriptors: halo slots of 18,432 B after 72 KB of
                // weights, A = slot + (7 + dx) x 16 B, K-step 2 x 2,304 B (LBO 2,304); B = weights + blk x 1,024
                // + dx x 24,576 + K-step x 2 x 3,072 (LBO 3,072).  5: as the layer; 6: A starts 128-byte aligned
                // (dx shift dropped); 7: as 5 with an LBO of 2,336 B (K-adjacent core matrices on different
                // banks); 8: as 5 with all A rows from one slot
                constexpr uint32_t i192 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(192 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t i128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t i64 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                constexpr uint32_t lbo = MODE == 7 ? 2336 : 2304;
                const uint32_t wb = s_u32(sm), sl = s_u32(sm) + 73728;
#pragma unroll
                for (int r = 0; r < 5; ++r) {
                    const uint32_t id = r == 0 ? i192 : (r < 3 ? i128 : i64);
                    // 10, 11: the two accumulator sets alternate by unit and a unit's first UMMA overwrites
                    const uint32_t dd = tmem + (MODE >= 10 ? (it & 1) * 192u : 0u) + (r == 2 ? 64u : (r == 4 ? 128u : 0u));
                    const int blk = r == 1 ? 1 : (r == 3 ? 2 : 0);
                    const uint32_t slot = sl + (MODE == 8 ? 0 : r) * 18432;
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint64_t au = sdesc(slot + (MODE == 6 ? 128 : (7 + dx) * 16) + 2 * j * lbo, lbo, 128);
                            const uint64_t bu = sdesc(wb + blk * 1024 + dx * 24576 + 2 * j * 3072, 3072, 128);
                            const uint32_t acc = (MODE >= 10 && r == 0 && dx == 0 && j == 0) ? 0u : 1u;
                            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dd), "l"(au), "l"(bu), "r"(id), "r"(acc));
                        }
                }
                if (MODE == 9 || MODE == 11)  // the unit's four commits (accumulators full, three slots free)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bars4[c])));
            } else {
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
#pragma unroll
                for (int u = 0; u < 6; ++u)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(s_u32(&bar)));
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int N, int MODE>
void run(int sms)
{
    long long* d;
    cudaMalloc(&d, 8);
    const int iters = 2000;
    const int smb = (MODE >= 5 ? 200 : 64) * 1024;
    cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    k<N, MODE><<<sms, 128, smb>>>(10, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<N, MODE><<<sms, 128, smb>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double mmas = (double)iters * (MODE == 4 ? 48 : (MODE >= 5 ? 60 : 8));
    const double flop = MODE == 4 ? 2.0 * 128 * 16 * (24 * 128 + 24 * 64) * iters * sms : 2.0 * 128 * N * 16 * mmas * sms;
    if (MODE >= 12) printf("rolling row mode %d: %.0f cycles per halo row\n", MODE, cyc / (double)iters);
    else if (MODE >= 5) printf("triple unit mode %d: %.0f cycles per unit of 60 UMMAs (model 3840)\n", MODE, cyc / (double)iters);
    printf("N=%3d mode=%d: %.1f cycles/MMA (%.0f per 48), %.0f TFLOP/s (err %s)\n", N, MODE, cyc / mmas, cyc / mmas * 48, flop / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, 12>(sms);
    run<64, 13>(sms);
    run<64, 14>(sms);
    run<64, 15>(sms);
    run<64, 5>(sms);
    run<64, 6>(sms);
    run<64, 7>(sms);
    run<64, 8>(sms);
    run<64, 9>(sms);
    run<64, 10>(sms);
    run<64, 11>(sms);
    run<16, 0>(sms);
    run<16, 1>(sms);
    run<32, 1>(sms);
    run<64, 4>(sms);
    run<64, 0>(sms);
    run<64, 1>(sms);
    run<64, 2>(sms);
    run<64, 3>(sms);
    run<128, 2>(sms);
    run<128, 3>(sms);
    run<192, 2>(sms);
    run<128, 0>(sms);
    run<128, 1>(sms);
    run<256, 0>(sms);
    run<256, 1>(sms);
    return 0;
}
