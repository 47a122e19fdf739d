// K5 row-unit layer timeline (k_conv64_tc2): builds cnn.cu with -DK5_TRACE (optionally -DK5_NO_STORE /
// -DK5_NO_TMA timing experiments), times whole denoises with CUDA events and prints, for the last middle
// layer, the median over CTAs of the per-CTA stamps and of the MMA issuer's cumulative stall cycles.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_1911_09278_b200/csrc/cnn.cuh"
namespace mace { void k5_trace_copy(long long* host); }
static long long med(std::vector<long long> v)
{
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}
int main()
{
    const int n = 512;
    mace::Cnn cnn;
    std::vector<uint16_t> w(64 * 9 + 15 * 64 * 64 * 9 + 64 * 9, 0x3c00);  // small bf16 values
    cnn.set_weights(w.data(), 17, 64);
    float *x, *y;
    cudaMalloc(&x, n * n * 4);
    cudaMalloc(&y, n * n * 4);
    cudaMemset(x, 0, n * n * 4);
    for (int r = 0; r < 5; ++r) cnn.apply(x, y, n, n, 0, 148, nullptr);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) cnn.apply(x, y, n, n, 0, 148, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms / 20);
    }
    printf("ms per 512^2 denoise (best of 5 x 20): %.4f\n", best);
    cudaDeviceSynchronize();
    static long long t[148][64];
    mace::k5_trace_copy(&t[0][0]);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    auto col = [&](int i, int base) {
        std::vector<long long> v;
        for (int c = 0; c < 144; ++c) v.push_back(t[c][i] - (base >= 0 ? t[c][base] : 0));  // CTAs with 14 rows
        return med(v);
    };
    printf("median over CTAs, cycles from CTA start: gdc wait passed %lld, weights seen by MMA warp %lld, end %lld\n",
           col(30, 0), col(1, 0), col(31, 0));
    for (int u = 0; u < 5; ++u)
        printf("  unit %d: issued %6lld  acc read %6lld  stored %6lld | cumulative stall: halo rows %6lld  acc free %6lld  in issue %6lld\n", u,
               col(2 + 2 * u, 0), col(3 + 2 * u, 0), col(50 + u, 0), col(32 + u, -1), col(40 + u, -1), col(56 + u, -1));
    printf("  unit 2 in detail (cycles from CTA start): before rows %lld | after row y+1 %lld, y %lld, y+2 %lld, y-1 %lld, y+3 %lld | after acc commit %lld, after slot commits %lld\n",
           col(18, 0), col(19, 0), col(20, 0), col(21, 0), col(22, 0), col(23, 0), col(24, 0), col(25, 0));
    long long s_mn = 1ll << 62, s_mx = 0, e_mn = 1ll << 62, e_mx = 0;
    for (int c = 0; c < 148; ++c) {
        s_mn = std::min(s_mn, t[c][48]);
        s_mx = std::max(s_mx, t[c][48]);
        e_mn = std::min(e_mn, t[c][49]);
        e_mx = std::max(e_mx, t[c][49]);
    }
    printf("globaltimer ns: CTA starts spread %lld, ends spread %lld, first start -> last end %lld, median CTA life %lld\n",
           s_mx - s_mn, e_mx - e_mn, e_mx - s_mn, col(49, 48));
    return 0;
}
