// kernels_tc.cuh — BF16 tcgen05 sampled-layer kernels (K2 fwd, K4 dgrad, K5 wgrad).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace bnn {

// K2 (mode 0) / K4 (mode 1): one CTA = 128 rows of the output feature dim (M) × up to 256
// batch rows (N) of one sample; A = W_s generated on chip, B = TMA (tmB: 3-D map
// [depth = sample][rows = batch][inner = reduction dim], box 64 × 256 × 1, SWIZZLE_128B).
struct TcGenArgs {
    SampledLayer L;
    SampleKeys kk;
    int mode;            // 0 fwd (M = L.N, R = L.K), 1 dgrad (M = L.K, R = L.N)
    int B;               // batch rows of a sample
    int b_shared;        // B operand is shared by all samples (layer-0 input)
    int M, R;
    int nb;              // MMA N: round_up(min(B, 256), 16)
    void* out;           // fwd: bf16 activations or fp32 logits; dgrad: bf16 gradients (fp32: out_f32)
    int64_t out_stride_s;
    int ldo;
    int out_f32, relu;
    const __nv_bfloat16* mask;  // dgrad: input activations of the layer (ReLU mask source)
    int64_t mask_stride_s;
    int ldm;
    int vec_ok;          // μ/σ rows are 16-byte aligned (float4 loads)
    float* dbpart;       // dgrad: fp32 column sums per 16-row chunk, [s][B/16][M]
    int64_t dbpart_stride_s;
    DropArgs drop;       // MC dropout: fwd masks the ReLU output, dgrad scales by 1/(1 − p)
    int mu_only;         // MC dropout: σ = 0, so W_s = RN_bf16(μ) without drawing ε
    const float* res_f32;  // fwd, out_f32: added to the output (same layout), or null
};
void launch_gen_gemm(const CUtensorMap& tmB, const TcGenArgs& a, int S, cudaStream_t st);
// the same with a second descriptor of the B operand in 128-row boxes: layers with R ≤ 768 and
// many rows per sample then run W-stationary with 128-row tiles (kernels_tc.cu)
void launch_gen_gemm_ws(const CUtensorMap& tmB256, const CUtensorMap& tmB128, const TcGenArgs& a, int S,
                        cudaStream_t st);

// K5: grouped over up to 4 layers; CTA = 128 n × kWgradTileK k tile, loops over all S samples.
constexpr int kMaxWgradLayers = 4;
constexpr int kWgradTileK = 112;  // multiple of 16 (MMA N), ≤ 128 (two 64-wide TMA blocks)
struct WgradLayer {
    SampledLayer L;
    int mtiles, ktiles, tile_base;
    int b_shared;
};
struct TcWgradArgs {
    int skip_eps;        // MC dropout: acc_ρ is not used, the epilogue draws no ε
    SampleKeys kk;
    int S, B;
    float scale;
    float* acc_mu;
    float* acc_rho;
    int nlayers;
    WgradLayer lay[kMaxWgradLayers];
    // row splits (many rows per sample, e.g. the ViT's tokens): split z of nsplit owns 64-row
    // blocks [z·per, …) of every sample and writes its scaled partials to part + part_off[layer]
    // as [z][μ|ρ][N·K]; launch_wgrad_tc then adds the splits in order (deterministic). nsplit ≤ 1:
    // the epilogue updates acc in place.
    int nsplit;
    float* part;
    int64_t part_off[kMaxWgradLayers];
};
struct TcWgradMaps {
    CUtensorMap g[kMaxWgradLayers];  // G_l: [S][B][N_l], box 64 × 64 × 1
    CUtensorMap x[kMaxWgradLayers];  // X_l: [S or 1][B][K_l], box 64 × 64 × 1
};
void launch_wgrad_tc(const TcWgradMaps& maps, const TcWgradArgs& a, cudaStream_t st);

}  // namespace bnn
