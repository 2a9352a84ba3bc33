// kernels_vit.cuh — launchers of the Bayesian ViT's non-GEMM kernels (kernels_vit.cu).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bnn {

// w[s][i] = μ[off + i] + σ[off + i]·ε_s(t, 0, i), i < n (1-D tensors: LayerNorm g/b, cls, pos)
void launch_vit_sample_vec(const float* mu, const float* sigma, int64_t off, uint32_t t, int n, const SampleKeys& kk,
                           int S, float* out, cudaStream_t st);
// P[s][b][patch][(dy·p + dx)·C + c] from x [B][H][W][C] (aug: per-sample crop + flip, docs/EPS.md §4)
void launch_vit_patchify(const float* x, int S, int B, int H, int W, int C, int p, int aug, uint64_t seed,
                         uint32_t step, uint32_t s0, int b_off, float* P, cudaStream_t st);
// X[s][b][t] = (t ? E[s][b][t−1] : cls_s) + pos_s[t]
void launch_vit_embed(const float* E, const float* cls, const float* pos, int S, int B, int T, int D, float* X,
                      cudaStream_t st);
// LayerNorm of `rows` rows per sample (row pitch ld, sample pitch sX); stats[s][row] = (mean, rstd)
void launch_vit_ln_fwd(const float* X, int S, int rows, int64_t ld, int64_t sX, int D, const float* g, const float* b,
                       float* Y, int64_t ldy, int64_t sY, float* stats, cudaStream_t st);
// dX (pitch ld, sX) += LayerNorm backward of dY; dyxh[s][row][D] = dY ⊙ x̂ (the g-gradient rows)
void launch_vit_ln_bwd(const float* dY, int64_t ldy, int64_t sdY, const float* X, int S, int rows, int64_t ld,
                       int64_t sX, int D, const float* g, const float* stats, float* dX, float* dyxh, cudaStream_t st);
// LayerNorm backward of all `rows` rows of each sample (pitch D) with the γ / β gradient sums of
// every 64-row chunk written to part_g / part_b [s][⌈rows/64⌉][D] (launch_bias_grad's parts) and,
// if dXb, a bf16 copy of the updated dX; if part_x, the chunk sums of the updated dX (the bias
// gradient source of the projection whose output gradient dX is); requires vit_ln_bwd_fused_ok(D)
bool vit_ln_bwd_fused_ok(int D);
void launch_vit_ln_bwd_fused(const float* dY, const float* X, int S, int rows, int D, const float* g,
                             const float* stats, float* dX, __nv_bfloat16* dXb, float* part_g, float* part_b,
                             float* part_x, cudaStream_t st);
// dUb = bf16(dA ⊙ GELU'(U)) and part[s][⌈rows/64⌉][M] = its fp32 64-row chunk sums (M % 4 == 0)
void launch_vit_gelu_bwd_fused(const float* U, const float* dA, int S, int rows, int M, __nv_bfloat16* dUb,
                               float* part, cudaStream_t st);
// softmax attention of every (head, example, sample): QKV [s][b][T][3D] → O [s][b][T][D], A [s][b][h][T][T]
void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, float* O, float* A, cudaStream_t st);
void launch_vit_attn_bwd(const float* QKV, const float* A, const float* dO, int S, int B, int T, int D, int heads,
                         float* dQKV, cudaStream_t st);
void launch_vit_gelu(const float* U, int64_t n, float* A, cudaStream_t st);
void launch_vit_gelu_bwd(const float* U, int64_t n, float* dA, cudaStream_t st);  // dA ⊙= GELU'(U)
void launch_vit_add(float* Y, const float* X, int64_t n, cudaStream_t st);       // Y += X
// out[s][b][k] = in[s][b][t0 + k], k < nt (token rows of width D, T per example)
// BF16 mode (the projections on tcgen05): bf16 outputs of the GEMM operands, bf16 inputs of
// the dgrad outputs
void launch_vit_patchify(const float* x, int S, int B, int H, int W, int C, int p, int aug, uint64_t seed,
                         uint32_t step, uint32_t s0, int b_off, __nv_bfloat16* P, cudaStream_t st);
void launch_vit_ln_fwd(const float* X, int S, int rows, int64_t ld, int64_t sX, int D, const float* g, const float* b,
                       __nv_bfloat16* Y, int64_t ldy, int64_t sY, float* stats, cudaStream_t st);
void launch_vit_ln_bwd(const __nv_bfloat16* dY, int64_t ldy, int64_t sdY, const float* X, int S, int rows, int64_t ld,
                       int64_t sX, int D, const float* g, const float* stats, float* dX, float* dyxh, cudaStream_t st);
void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, __nv_bfloat16* O, float* A,
                         cudaStream_t st);
void launch_vit_attn_bwd(const float* QKV, const float* A, const __nv_bfloat16* dO, int S, int B, int T, int D,
                         int heads, float* dQKV, cudaStream_t st);
// the BF16 step's backward with an fp32 dO (products in TF32 on the warp MMA, as the bf16 overloads)
void launch_vit_attn_bwd_tf32(const float* QKV, const float* A, const float* dO, int S, int B, int T, int D,
                              int heads, float* dQKV, cudaStream_t st);
void launch_vit_gelu(const float* U, int64_t n, __nv_bfloat16* A, cudaStream_t st);
void launch_vit_gelu_bwd(const float* U, int64_t n, const __nv_bfloat16* dA, float* dU, __nv_bfloat16* dUb,
                         cudaStream_t st);
void launch_vit_cast_bf16(const float* x, int64_t n, __nv_bfloat16* y, cudaStream_t st);
// dA ⊙= GELU'(U) in place, and its bf16 copy
void launch_vit_gelu_bwd_cast(const float* U, int64_t n, float* dA, __nv_bfloat16* dUb, cudaStream_t st);
void launch_vit_widen(const __nv_bfloat16* x, int64_t n, float* y, cudaStream_t st);
void launch_vit_gather_tokens(const float* in, int S, int B, int T, int t0, int nt, int D, float* out,
                              cudaStream_t st);

}  // namespace bnn
