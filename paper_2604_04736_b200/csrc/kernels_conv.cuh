// kernels_conv.cuh — sampled convolution kernels of the ResNet-18-shaped CNN (C3–C5).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bnn {

// Geometry of one convolution over a batch of B NHWC images (per sample).
struct ConvShape {
    int B, H, W, C;      // input
    int OH, OW, CO;      // output
    int k, stride, pad;  // square kernel
};

void launch_conv_fwd_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                          const float* X, int64_t sX, const float* R, int64_t sR, float* Y,
                          int64_t sY, bool relu, cudaStream_t st);
void launch_conv_dgrad_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                            const float* G, int64_t sG, float* dX, int64_t sdX, bool accumulate,
                            cudaStream_t st);
void launch_conv_wgrad_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                            const float* G, int64_t sG, const float* X, int64_t sX, float scale,
                            float* acc_mu, float* acc_rho, cudaStream_t st);
void launch_relu_mask(float* g, const float* y, int64_t n, cudaStream_t st);
void launch_add(float* dst, const float* src, int64_t n, cudaStream_t st);
void launch_gap_fwd(const float* y, int R, int HW, int C, float* out, cudaStream_t st);
void launch_gap_bwd(const float* gpool, int R, int HW, int C, float* gy, cudaStream_t st);
void launch_augment(const float* x, int S, int B, int H, int W, int C, uint64_t seed,
                    uint32_t step, uint32_t s0, int b_off, float* out, cudaStream_t st);

}  // namespace bnn
