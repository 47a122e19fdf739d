// K5 rolling-accumulator layer timeline (k_conv64_roll): cnn.cu built with -DK5_TRACE.
#include <algorithm>
#include <array>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_1911_09278_b200/csrc/cnn.cuh"
namespace mace { void k5_trace_copy(long long* host); unsigned k5_life_copy(long long* host, bool reset); }
static long long med(std::vector<long long> v)
{
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}
int main()
{
    const int n = 512;
    mace::Cnn cnn;
    std::vector<uint16_t> w(64 * 9 + 15 * 64 * 64 * 9 + 64 * 9, 0x3c00);
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
    printf("ms per 512^2 denoise (best of 5 x 20): %.4f  (err %s)\n", best, cudaGetErrorString(cudaGetLastError()));
    cudaDeviceSynchronize();
#ifdef K5_TRACE
    static long long t[148][64];
    mace::k5_trace_copy(&t[0][0]);
    auto col = [&](int i, int base) {
        std::vector<long long> v;
        for (int c = 0; c < 144; ++c) v.push_back(t[c][i] - (base >= 0 ? t[c][base] : 0));
        return med(v);
    };
    printf("gdc wait passed %lld, first halo row landed %lld, ", col(30, 0), col(31, 0));
    printf("weights seen %lld\nhalo row committed (cycles from CTA start):", col(1, 0));
    for (int q = 0; q < 16; ++q) printf(" %lld", col(2 + q, 0));
    printf("\noutput row read by the epilogue:");
    for (int q = 0; q < 14; ++q) printf(" %lld", col(32 + q, 0));
    printf("\ncumulative issuer waits (halo + accumulator) after row:");
    for (int q = 0; q < 14; ++q) printf(" %lld", col(50 + q, -1));
    printf("\nissuer totals: halo wait %lld, accumulator wait %lld, in issue (fast rows) %lld, in commits %lld, in issue (wrap rows) %lld\n", col(18, -1),
           col(19, -1), col(20, -1), col(21, -1), col(22, -1));
    printf("median CTA life %lld ns\n", col(49, 48));
    {   // one denoise alone: per-SM chains of CTA lives (globaltimer)
        static long long life[4096][4];
        mace::k5_life_copy(&life[0][0], true);
        cnn.apply(x, y, n, n, 0, 148, nullptr);
        cudaDeviceSynchronize();
        const unsigned cnt = mace::k5_life_copy(&life[0][0], false);
        std::vector<std::vector<std::array<long long, 3>>> per(256);
        for (unsigned i = 0; i < cnt && i < 4096; ++i) per[life[i][0]].push_back({life[i][1], life[i][2], life[i][3]});
        std::vector<long long> gaps, lifes, waits, periods;
        for (auto& v : per) {
            std::sort(v.begin(), v.end());
            for (size_t i = 0; i + 1 < v.size(); ++i) {
                gaps.push_back(v[i + 1][0] - v[i][2]);
                periods.push_back(v[i + 1][0] - v[i][0]);
            }
            for (auto& r : v) {
                lifes.push_back(r[2] - r[0]);
                waits.push_back(r[1] - r[0]);
            }
        }
        printf("%u CTA records: median life %lld ns, start -> gdc wait passed %lld ns, end -> next start on the SM %lld ns, start -> next start %lld ns\n",
               cnt, med(lifes), med(waits), med(gaps), med(periods));
    }
#endif
    return 0;
}
