// Microbenchmark: does the K5 pair-unit UMMA stream (2 x 12 N=128 + 2 x 12 N=64, kind::f16, SS,
// SWIZZLE_NONE) slow down when other warps read TMEM (the epilogue's tcgen05.ld) or when bulk
// copies fill shared memory (the TMA halo rows) at the same time?  One CTA per SM.
//   mode 0: UMMAs alone; 1: + two warps streaming tcgen05.ld 32x32b.x16 from other TMEM columns;
//   2: + one thread streaming 18 KB cp.async.bulk copies into shared memory; 3: both.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out, const unsigned char* gsrc)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, cbar;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tslot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&cbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        stop = 0;
    }
    for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 32) {
        constexpr uint32_t i128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        constexpr uint32_t i64 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t a = sdesc(s_u32(sm), 144 * 16, 128);
        const uint64_t b = sdesc(s_u32(sm + 24576), 192 * 16, 128);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 48; ++u) {
                const uint32_t id = u < 24 ? i128 : i64;
                const uint32_t dd = tmem + (u >= 36 ? 64u : 0u);
                const uint64_t au = a + (uint64_t)((((u % 3) * 16) + ((u / 3) % 4) * 2 * 144 * 16) >> 4);
                const uint64_t bu = b + (uint64_t)((((u / 3) % 4) * 2 * 192 * 16) >> 4);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dd), "l"(au), "l"(bu), "r"(id));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(s_u32(&bar)));
        long long t1 = clock64();
        stop = 1;
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if ((MODE & 1) && warp >= 2) {  // TMEM readers on their own lane quadrant, columns 256..511
        uint32_t acc = 0;
        while (!stop) {
            uint32_t r[16];
            const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + 256u + (uint32_t)((acc & 15) * 16);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(base));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 16; ++i) acc += r[i];
        }
        if (acc == 0x12345678u) out[1] = acc;
    } else if ((MODE & 2) && threadIdx.x == 0) {  // bulk copies of 18 KB into shared memory, back to back
        uint32_t phase = 0;
        while (!stop) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&cbar)), "r"(18432u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             s_u32(sm + 40960)), "l"(gsrc + (size_t)blockIdx.x * 18432), "r"(18432u), "r"(s_u32(&cbar))
                         : "memory");
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(ok) : "r"(s_u32(&cbar)), "r"(phase));
            phase ^= 1;
        }
    }
    (void)lane;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int MODE>
void run(int sms, const unsigned char* gsrc)
{
    long long* d;
    cudaMalloc(&d, 16);
    const int iters = 400;
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE><<<sms, 128, smem>>>(10, d, gsrc);
    k<MODE><<<sms, 128, smem>>>(iters, d, gsrc);
    cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %.0f cycles per 48-UMMA pair unit (err %s)\n", MODE, (double)cyc / iters,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned char* g;
    cudaMalloc(&g, (size_t)sms * 18432);
    cudaMemset(g, 0, (size_t)sms * 18432);
    run<0>(sms, g);
    run<1>(sms, g);
    run<2>(sms, g);
    run<3>(sms, g);
    return 0;
}
