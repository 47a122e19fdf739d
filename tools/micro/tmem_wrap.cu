// Does a UMMA's D region wrap around the 512 TMEM columns?  One CTA: A = ones (128 x 16), B = ones (192 x 16),
// D = A B^T (N = 192, overwrite) at column 448 of a 512-column allocation; then columns 0..127 and 448..511 are
// read back (16.0 where the UMMA wrote, the 7.0 fill elsewhere).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__global__ void __launch_bounds__(128, 1) k(float* out, int dcol)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tslot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(sm);
    for (int i = threadIdx.x; i < 32 * 1024 / 2; i += blockDim.x) h[i] = __float2bfloat16(1.0f);
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    // fill all 512 columns with 7.0
    for (int c = 0; c < 512; ++c) {
        const uint32_t v = __float_as_uint(7.0f);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 32) {
        constexpr uint32_t i192 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(192 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t a = sdesc(s_u32(sm), 128 * 16, 128);           // K-major, core matrices 8 rows x 16 B, LBO = 128 rows x 16 B
        const uint64_t b = sdesc(s_u32(sm + 8192), 192 * 16, 128);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)dcol), "l"(a), "l"(b), "r"(i192));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)));
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(s_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < 512; ++c) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (lane == 0 && warp == 0) out[c] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}
int main()
{
    float* d;
    cudaMalloc(&d, 512 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int dcol : {64, 448}) {
        k<<<1, 128, 64 * 1024>>>(d, dcol);
        cudaError_t e = cudaDeviceSynchronize();
        float h[512];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("D at column %d (err %s): written columns:", dcol, cudaGetErrorString(e));
        int run0 = -1;
        for (int c = 0; c <= 512; ++c) {
            const bool w = c < 512 && h[c] == 16.0f;
            if (w && run0 < 0) run0 = c;
            if (!w && run0 >= 0) {
                printf(" [%d, %d)", run0, c);
                run0 = -1;
            }
        }
        printf("  (col 0 = %.1f, col 511 = %.1f)\n", h[0], h[511]);
        if (e != cudaSuccess) break;
    }
    return 0;
}
