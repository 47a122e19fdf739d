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
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tslot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
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
    cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<N, MODE><<<sms, 128, 64 * 1024>>>(10, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<N, MODE><<<sms, 128, 64 * 1024>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double mmas = (double)iters * (MODE == 4 ? 48 : 8);
    const double flop = MODE == 4 ? 2.0 * 128 * 16 * (24 * 128 + 24 * 64) * iters * sms : 2.0 * 128 * N * 16 * mmas * sms;
    printf("N=%3d mode=%d: %.1f cycles/MMA (%.0f per 48), %.0f TFLOP/s (err %s)\n", N, MODE, cyc / mmas, cyc / mmas * 48, flop / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
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
