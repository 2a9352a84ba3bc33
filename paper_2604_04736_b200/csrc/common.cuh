// common.cuh — small shared device/host helpers of libbnn (no method arithmetic here).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace bnn {

constexpr int kNumSMs = 148;  // B200

// cudaFuncAttributeMaxDynamicSharedMemorySize of kernel `func` on the current device, set once
// per (kernel, device) — the attribute is per device, and launchers may run from several host
// threads (round-1 ADVICE: a function-static flag skipped a second device and raced). Defined in
// kernels_simt.cu.
void ensure_smem_attr(const void* func, int bytes);

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Pack two fp32 into a bf16x2 word (round to nearest even), low half = a.
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// softplus(ρ) = max(ρ,0) + log1p(e^{-|ρ|}), σ parameterisation of DESIGN.md R1.
__device__ __forceinline__ float softplus_f(float r) {
    return fmaxf(r, 0.0f) + log1pf(expf(-fabsf(r)));
}
__device__ __forceinline__ float sigmoid_f(float r) {
    if (r >= 0.0f) return 1.0f / (1.0f + expf(-r));
    const float e = expf(r);
    return e / (1.0f + e);
}
// ln σ with the log-domain branch for very negative ρ (R4)
__device__ __forceinline__ float log_sigma_f(float r, float sigma) {
    return r < -15.0f ? r - 0.5f * expf(r) : logf(sigma);
}

}  // namespace bnn
