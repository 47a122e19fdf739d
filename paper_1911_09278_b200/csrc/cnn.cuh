// K5 denoiser host object (see cnn.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>

namespace mace {

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count)
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) {
            p = nullptr;
            n = 0;
            throw std::runtime_error("cudaMalloc failed (denoiser buffers)");
        }
    }
    ~DevBuf()
    {
        if (p) cudaFree(p);
    }
};

// 3x3 weights of the 1-channel end layers, [tap 9][64] fp32 holding bf16 values; passed to the
// kernels by value (__grid_constant__), so every FMA reads its weight straight from the constant bank
struct ConvW9 {
    float v[9 * 64];
};

struct Cnn {
    bool ready = false;
    int H = 0, W = 0, Wp = 0;  // Wp: activation row pitch (W rounded up to 8 pixels)
    ConvW9 w_first{}, w_last{};          // layers 1 and 17
    DevBuf<__nv_bfloat16> w_mid;         // [15][9 taps][8 ic-groups][64 oc][8 ic]
    DevBuf<__nv_bfloat16> w_mid2;        // row-pair layout: [15][3 dx][8 ic-groups][dy2 | dy1 | dy0][64 oc][8 ic]
    int rows_unit = 2;                   // output rows per MMA unit (k_conv64_tc2<2|3>; 1 = k_conv64_tc), MACE_K5_ROWS
    DevBuf<__nv_bfloat16> w_last_tc;     // layer 17 for k_conv_last_tc: [9 taps][8 ic-groups][16 oc][8 ic]
    bool last_tc = true;                 // layer 17 on the tensor cores (MACE_K5_LAST=fma: CUDA cores)
    DevBuf<__nv_bfloat16> w_last_roll;   // layer 17 for k_conv_last_roll: [dx][ic-group][dy2 | dy1 | dy0 x 16 oc][8 ic]
    bool last_roll = true;               // ... with rolling accumulators (MACE_K5_LAST=tc: one UMMA run per output row)
    bool seq = false;                    // layers 2..16 in one persistent launch (MACE_K5_SEQ=1; slower)
    DevBuf<int> flags;                   // per-CTA layer-done flags of k_conv64_seq
    int epoch = 0;                       // flag epoch (one per persistent launch)
    bool seq_pipe = false;               // layers 2..16 as one pipelined persistent launch (MACE_K5_SEQ=2)
    DevBuf<int> pflags;                  // k_conv64_pipe: published row counts [cta][epilogue warp]
    int pipe_epoch = 0;
    int roll_epoch = 0;                  // persistent rolling-accumulator launches so far at this geometry
    DevBuf<__nv_bfloat16> act0, act1;    // channel-blocked [8 groups][H][Wp][8 ch]
    CUtensorMap map0{}, map1{};
    // weights: 17 layers in PyTorch OIHW order, bf16 bits, concatenated
    void set_weights(const uint16_t* bf16, int layers, int channels);
    void ensure(int h, int w);
    // out = x - net(x) for an h x w fp32 image (device pointers), on stream s
    void apply(const float* x, float* out, int h, int w, cudaStream_t s, int num_sms, int* launches);
    // one middle layer l (0..14 = layers 2..16) alone on a bf16 CHW input (host arrays; tests)
    void layer(int l, const uint16_t* in_chw, uint16_t* out_chw, int h, int w, cudaStream_t s, int num_sms);
    void launch_mid(int l, const CUtensorMap& m, __nv_bfloat16* dst, cudaStream_t s, int num_sms, bool pdl);
};

}  // namespace mace
