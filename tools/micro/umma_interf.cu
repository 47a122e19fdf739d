// Microbenchmark: does the K5 pair-unit UMMA stream (2 x 12 N=128 + 2 x 12 N=64, kind::f16, SS,
// SWIZZLE_NONE) slow down when other warps read TMEM (the epilogue's tcgen05.ld) or when bulk
// copies fill shared memory (the TMA halo rows) at the same time?  One CTA per SM.
//   mode 0: UMMAs alone; 1: + two warps streaming tcgen05.ld 32x32b.x16 from other TMEM columns;
//   2: + one thread streaming 18 KB cp.async.bulk copies into shared memory; 3: both;
//   4: three tcgen05.commit per unit (as the layer issues); 5: one commit per unit;
//   6: the layer's issue path (whole warp, one asm block of 12 UMMAs per halo row); 7: 6 + five
//   mbarrier waits per unit.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

constexpr uint32_t kI128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr uint32_t kI64 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ void umma_row12(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t accumulate)
{
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

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out, const unsigned char* gsrc)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, cbar, dbar[3];
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tslot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&cbar)));
        for (int c = 0; c < 3; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&dbar[c])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        stop = 0;
    }
    for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (MODE >= 6 && warp == 1) {  // the layer's issue path: whole warp, row12 asm blocks, mbarrier waits
        const uint64_t a = sdesc(s_u32(sm), 144 * 16, 128);
        const uint64_t b = sdesc(s_u32(sm + 24576), 192 * 16, 128);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE == 7)
                for (int w = 0; w < 5; ++w) {  // completed barriers (phase 1 is the completed parity of a fresh barrier)
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\nselp.u32 %0, 1, 0, p;\n}\n"
                                     : "=r"(ok) : "r"(s_u32(&dbar[w % 3])));
                }
            umma_row12(tmem, a, b + (1024 >> 4), kI128, 0u);
            umma_row12(tmem, a + (2048 >> 4), b, kI128, 1u);  // (other "rows": shifted starts, same extent)
            umma_row12(tmem, a + (4096 >> 4), b + (2048 >> 4), kI64, 1u);
            umma_row12(tmem + 64, a + (6144 >> 4), b, kI64, 1u);
        }
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(s_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(s_u32(&bar)));
        long long t1 = clock64();
        if (lane == 0) {
            stop = 1;
            if (blockIdx.x == 0) out[0] = t1 - t0;
        }
    } else if (MODE < 6 && threadIdx.x == 32) {
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
            if (MODE >= 4)  // the layer's per-unit commits (accumulator ready, two halo rows free)
                for (int c = 0; c < (MODE == 4 ? 3 : 1); ++c)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&dbar[c])));
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
                             s_u32(sm + 102400)), "l"(gsrc + (size_t)blockIdx.x * 18432), "r"(18432u), "r"(s_u32(&cbar))
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
    const int smem = 128 * 1024;  // A at 0, B (the layer's 72 KB weight layout) at 24 KB, bulk-copy scratch at 100 KB
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
    run<4>(sms, g);
    run<5>(sms, g);
    run<6>(sms, g);
    run<7>(sms, g);
    return 0;
}
