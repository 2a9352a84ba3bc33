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

// ====================================================================== BF16 tcgen05 path
#include <cuda.h>
#include <cuda_bf16.h>

namespace bnn {

// W_s of one layer for Sc samples, bf16 [s][CO][K_pad]; column kp = tap·C_pad + ci (zero
// where ci ≥ C or tap ≥ k·k). The scratch of ONE layer for the current sample chunk: the
// weight reuse of a convolution (every element feeds B·OH·OW ≥ 2 K pixels) is spread over
// many CTAs, so W_s is formed once per (sample, layer, pass) into this L2-resident buffer
// instead of per pixel tile.
void launch_gen_wscratch(const SampledLayer& L, const SampleKeys& kk, int S, int C, int C_pad,
                         int taps, int K_pad, __nv_bfloat16* out, float* bias_out, cudaStream_t st);

// Persistent swap-AB conv (kernels_conv2.cu): M = 128 pixels, N = n_tile channels.
struct Conv2Args {
    int S;
    int B, H, W, C, C_pad;  // conv input per sample (C_pad = channel pitch of the input buffer)
    int OH, OW, CO;
    int k, stride, pad;
    int K_pad;              // W scratch row pitch
    int n_tile;             // 64, 128 or 256
    int tma_a;              // stride 1: A window by 5-D TMA (amap, 128-pixel box)
    const __nv_bfloat16* src;  // gathered A: fwd input [s][B][H][W][C_pad], dgrad dY [s][B][OH][OW][CO]
    int64_t src_stride_s;      // 0 ⇒ the input is shared by all samples
    __nv_bfloat16* out;        // fwd [s][B][OH][OW][CO]; dgrad [s][B][H][W][C]
    int64_t out_stride_s;      // also the stride of res / addsrc / mask
    const float* bias;         // fwd: sampled biases [S][CO]
    const __nv_bfloat16* res;  // fwd residual
    const __nv_bfloat16* addsrc;  // dgrad: other contribution, added before the mask
    const __nv_bfloat16* mask;    // dgrad: ReLU mask source (the conv input activation)
    int relu;
    float* bpart;              // dgrad: fp32 bias partials [s][parts][C]
    int64_t bpart_stride_s;
    int dbg;                   // timing experiments only (BNN_CONV_DEBUG); 0 in production
    uint32_t* mbits_out;       // fwd (relu): ReLU bitmask of the stored output, bit j of word
                               //   [pixel][c/32] = (stored bf16 of channel c > 0); or null
    const uint32_t* mbits;     // dgrad: bitmask of the layer input (replaces `mask` when set)
    const __nv_bfloat16* wsrc; // stem kernel: the layer's W scratch slot [s][CO][K_pad]
    int halo;                  // conv3, stride-1 3×3, 64-channel B operand: padded-stream tiles with
                               //   one halo window per tile (bmap = 1-row box of W + 2 pixels)
};
void launch_conv2_fwd(const CUtensorMap& amap, const CUtensorMap& wmap, const Conv2Args& a, cudaStream_t st);
void launch_conv2_dgrad(const CUtensorMap& amap, const CUtensorMap& wmap, const Conv2Args& a, cudaStream_t st);
int conv2_dgrad_parts(const Conv2Args& a);
// conv3: M = 128 output channels (weights: fwd W scratch K-major map, box 64 × 64; dgrad the
// transposed 4-D map, box 64 × 1 × 64 × 1), N = 256 pixels (tma_a: 5-D 256-pixel window map,
// else cp.async gather). For layers with ≤ 128 output channels.
void launch_conv3_fwd(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st);
void launch_conv3_dgrad(const CUtensorMap& wmapT, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st);
int conv3_dgrad_parts(const Conv2Args& a);
int conv3_halo_ok(int H, int W);
// conv64 (kernels_conv64.cu): stride-1 3×3 64 → 64-channel convs, W-stationary (the sample's 9
// tap blocks resident in shared memory, loaded once per CTA and sample) and tap-paired (6 MMA
// groups per 255-pixel tile of the padded stream); wmap = the 64-row K-major W map (fwd) or the
// transposed map (dgrad), bmap = the HALO window map. Bias partials: conv64_parts per sample.
struct Conv64RowMaps;
void launch_conv64_fwd(const CUtensorMap& wmap, const Conv64RowMaps& rows, const Conv2Args& a, cudaStream_t st);
void launch_conv64_dgrad(const CUtensorMap& wmapT, const Conv64RowMaps& rows, const Conv2Args& a, cudaStream_t st);
int conv64_parts(const Conv2Args& a);
int conv64_ok(int H, int W);
// stem (kernels_stem.cu): 3×3 stride-1 conv of the 8-channel input to 64 channels, pixels on M and two
// taps per MMA (SWIZZLE_NONE K-major operands, the taps' distance as the leading byte offset);
// xmap = 1-row (W + 2)-pixel boxes of the input, no swizzle; a.wsrc = the W scratch slot
struct StemRowMaps {  // boxes of 1 … 8 padded rows of the stem input
    CUtensorMap x[8];
};
void launch_stem_fwd(const StemRowMaps& xmaps, const Conv2Args& a, cudaStream_t st);
int stem_fwd_ok(const Conv2Args& a);
int stem_row_pitch(int W);  // padded-row length of the stem window (the map box width)
// conv64 weight gradient: the fp32 per-sample partials part[s][split][64][576] of the ε combine,
// one CTA per (sample, split) (nsplit = conv64_wgrad_nsplit(S)); ymap / xmap = the HALO window
// maps of dY and of the layer input.
struct ConvWgradArgs;
// Runs of padded rows loaded by one TMA op each: maps of box height h + 1 (h < 8) over dY and X
// (a run never crosses an image: its separator row is the box's out-of-range row).
struct Conv64RowMaps {
    CUtensorMap y[8], x[8];
};
void launch_conv64_wgrad(const Conv64RowMaps& maps, const ConvWgradArgs& a, cudaStream_t st);
int conv64_wgrad_ok(int H, int W);
int conv64_wgrad_nsplit(int S);
// ε-fused form (clusters of the S ≤ 8 samples of a split): writes scale·Σ_s (D_s, ε_s ⊙ D_s) to
// split partials part[split][μ | ρ][64·576] for launch_wgrad_split_reduce; nsplit =
// conv64_wgrad_eps_nsplit(S) (co-resident clusters, 0 = not available). Returns 0 or -1 (launch refused).
int conv64_wgrad_eps_nsplit(int S, int Gc);
int conv64_wgrad_eps_cluster(int S);  // default cluster size (BNN_WGRAD_EPS_CLUSTER overrides)
int launch_conv64_wgrad_eps(const Conv64RowMaps& maps, const ConvWgradArgs& a, cudaStream_t st);


struct ConvWgradArgs {
    SampledLayer L;
    SampleKeys kk;
    int S;
    int B, H, W, C, C_pad, OH, OW, CO, k, stride, pad;
    const __nv_bfloat16* X;  // conv input [s][B][H][W][C_pad]
    int64_t X_stride_s;
    float scale;
    float* part;             // conv2 wgrad: [s][split][CO][cols] fp32 per-sample partials (unscaled);
                             // SIMT wgrad: [nsplit][2][CO·k·k·C] (μ then ρ), scaled
    int nsplit;
    int tma_b;               // stride 1: X window by 5-D TMA (xmap: 64 ci × kpx pixels × channel blocks)
    int n_tile;              // conv2 wgrad: column-tile width (256; the last tile may be narrower)
    int kpx;                 // pixels per k-step: 128 on the TMA path where the window fits, else 64
    int dbg;                 // timing experiments only (BNN_CONV_DEBUG); 0 in production
    int eps_cluster;         // ε-fused conv64 wgrad: samples per thread-block cluster (divides S, ≤ 8)
    int cps;                 // conv2 wgrad: CTAs per SM (2 needs kpx = 64)
};
void launch_wgrad_split_reduce(const float* part, int nsplit, int64_t n, int64_t off,
                               float* acc_mu, float* acc_rho, cudaStream_t st);
// conv2 wgrad, phase 1 (tensor cores): per-sample, per-pixel-split weight gradients
//   part[s][split][co][tap·C + ci] = Σ_{pix ∈ split} dY_s[pix][co] · X_s[pix ⊕ tap][ci]   (fp32)
// phase 2 (ALU): acc_μ += scale·Σ_s Σ_split part;  acc_ρ += scale·Σ_s ε_s ⊙ Σ_split part.
void launch_conv2_wgrad(const CUtensorMap& gmap, const CUtensorMap& xmap, const ConvWgradArgs& a,
                        cudaStream_t st);
void launch_wgrad_eps_combine(const SampledLayer& L, const SampleKeys& kk, int S, int nsplit, int CO,
                              int Kt, const float* part, float scale, float* acc_mu, float* acc_rho,
                              cudaStream_t st);
void launch_wgrad_eps_combine_stem(const SampledLayer& L, const SampleKeys& kk, int S, int nsplit, int CO, int taps,
                                   int C, int Ktp, const float* part, float scale, float* acc_mu, float* acc_rho,
                                   cudaStream_t st);
int conv2_wgrad_ntile(int Kt);
int conv2_wgrad_cps();
int conv2_wgrad_nsplit(int base, int blocks, int cps = 1);
// partial columns: taps·C, or (stem, C_pad < 64) ⌈taps/8⌉·64
inline int conv2_wgrad_cols(int taps, int C, int C_pad) { return C_pad < 64 ? ((taps + 7) / 8) * 64 : taps * C; }

// image-path helpers on bf16 NHWC buffers
void launch_input_bf16(const float* x, int S, int B, int H, int W, int C, int C_pad, int aug,
                       uint64_t seed, uint32_t step, uint32_t s0, int b_off, __nv_bfloat16* out,
                       cudaStream_t st);
void launch_gap_fwd_bf16(const __nv_bfloat16* y, int R, int HW, int C, __nv_bfloat16* out,
                         cudaStream_t st);
// gy[r][hw][c] = mask(y > 0)·gpool[r][c]/HW (bf16) and part[r][c] = Σ_hw gy (fp32)
void launch_gap_bwd_bf16(const __nv_bfloat16* gpool, int ldg, const __nv_bfloat16* y, int R,
                         int HW, int C, __nv_bfloat16* gy, float* part, cudaStream_t st);
// stem / generic small wgrad on bf16 operands (SIMT): same math as launch_conv_wgrad_fp32
void launch_conv_wgrad_simt_bf16(const SampledLayer& L, const SampleKeys& kk, int S,
                                 const ConvShape& c, int C_pad, const __nv_bfloat16* G,
                                 int64_t sG, const __nv_bfloat16* X, int64_t sX, float scale,
                                 float* part, int nsplit, cudaStream_t st);

}  // namespace bnn
