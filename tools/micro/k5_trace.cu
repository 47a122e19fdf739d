// K5 layer timeline: builds cnn.cu with -DK5_TRACE and prints per-CTA clock64 stamps of one layer.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_1911_09278_b200/csrc/cnn.cuh"
namespace mace { void k5_trace_copy(long long* host); }
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
    for (int r = 0; r < 3; ++r) cnn.apply(x, y, n, n, 0, 148, nullptr);
    cudaDeviceSynchronize();
    static long long t[148][64];
    mace::k5_trace_copy(&t[0][0]);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    for (int c : {0, 1, 73, 147}) {
        long long t0 = t[c][0];
        printf("cta %3d: weights %lld |", c, t[c][1] - t0);
        for (int k = 0; k < 14; ++k) printf(" mma%d %lld epi %lld", k, t[c][2 + 2 * k] - t0, t[c][3 + 2 * k] - t0);  // units (pairs by default)
        printf("\n   tma issue:");
        for (int q = 0; q < 16; ++q) printf(" %lld", t[c][32 + q] - t0);
        printf("\n   row landed:");
        for (int q = 2; q < 16; ++q) printf(" %lld", t[c][48 + q] - t0);
        printf("\n");
    }
    long long mn = t[0][0], mx = 0;
    for (int c = 0; c < 148; ++c) { if (t[c][0] < mn) mn = t[c][0]; if (t[c][3 + 2 * 13] > mx) mx = t[c][3 + 2 * 13]; }
    printf("span start..last epilogue: %lld cycles\n", mx - mn);
    return 0;
}
