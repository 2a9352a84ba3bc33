// kernels_vit.cu — the non-GEMM kernels of the Bayesian ViT step (
// PAPER.md:305-315): patch extraction with the per-sample crop/flip, token assembly with the
// sampled cls / position embeddings, LayerNorm, softmax attention, GELU and their backward
// passes. The sampled projections (patch embedding, QKV, output projection, MLP, head) run on
// the sampled-layer GEMM kernels shared with the MLP (kernels_simt.cu FP32 / kernels_tc.cu BF16).
//
// Layout: token rows [s][b][t][·] (t = 0 the cls token), fp32. LayerNorm and attention follow
// oracle/vit_oracle.c's definitions (LN eps 1e-6 with the biased variance; scores / √dh;
// exact-erf GELU) — written independently, no shared code.
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels_vit.cuh"

namespace bnn {

__device__ __forceinline__ float ldf(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void stf(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void stf(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }
// exact-erf GELU and its derivative (R29)
__device__ __forceinline__ float gelu_f(float u) { return 0.5f * u * (1.0f + erff(u * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_df(float u) {
    return 0.5f * (1.0f + erff(u * 0.70710678118654752f)) + u * 0.39894228040143268f * __expf(-0.5f * u * u);
}

// ------------------------------------------------------------------------ sampled vectors
// w[s][i] = μ[off + i] + σ[off + i]·ε(t, 0, i) for the 1-D tensors (LayerNorm g/b, cls, pos)
__global__ void vit_sample_vec_kernel(const float* __restrict__ mu, const float* __restrict__ sigma, int64_t off,
                                      uint32_t t, int n, SampleKeys kk, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, s = blockIdx.y;
    if (i >= n) return;
    out[(int64_t)s * n + i] = __fmaf_rn(sigma[off + i], eps1(kk.key, kk.step, kk.s0 + s, t, 0u, (uint32_t)i), mu[off + i]);
}

void launch_vit_sample_vec(const float* mu, const float* sigma, int64_t off, uint32_t t, int n, const SampleKeys& kk,
                           int S, float* out, cudaStream_t st) {
    vit_sample_vec_kernel<<<dim3((n + 255) / 256, S), 256, 0, st>>>(mu, sigma, off, t, n, kk, out);
}

// ------------------------------------------------------------------------ patches
// P[s][b][pi][(dy·p + dx)·C + c] of the (crop + flip augmented, docs/EPS.md §4) image b
template <class TO>
__global__ void vit_patchify_kernel(const float* __restrict__ x, int B, int H, int W, int C, int p, int aug,
                                    EpsKey key, uint32_t step, uint32_t s0, int b_off, TO* __restrict__ P) {
    const int b = blockIdx.x, s = blockIdx.y;
    int dx = 4, dy = 4, flip = 0;
    if (aug) {
        const uint4 y = philox10(make_uint4(0u, (uint32_t)(b_off + b), (4095u << 20) | (s0 + s), step), key);
        dx = (int)(y.x % 9u);
        dy = (int)(y.y % 9u);
        flip = (int)(y.z & 1u);
    }
    const float* src = x + (int64_t)b * H * W * C;
    const int pw = W / p, pk = p * p * C, np = (H / p) * pw;
    TO* dst = P + ((int64_t)s * B + b) * np * pk;
    for (int i = threadIdx.x; i < np * pk; i += blockDim.x) {
        const int pi = i / pk, e = i - pi * pk;
        const int c = e % C, q = e / C, ddx = q % p, ddy = q / p;
        const int r = (pi / pw) * p + ddy, cc = (pi % pw) * p + ddx;
        const int jj = flip ? W - 1 - cc : cc;
        const int si = r + dy - 4, sj = jj + dx - 4;
        stf(dst, i, (si >= 0 && si < H && sj >= 0 && sj < W) ? src[((int64_t)si * W + sj) * C + c] : 0.0f);
    }
}

void launch_vit_patchify(const float* x, int S, int B, int H, int W, int C, int p, int aug, uint64_t seed,
                         uint32_t step, uint32_t s0, int b_off, float* P, cudaStream_t st) {
    vit_patchify_kernel<float><<<dim3(B, S), 256, 0, st>>>(x, B, H, W, C, p, aug, make_key(seed), step, s0, b_off, P);
}
void launch_vit_patchify(const float* x, int S, int B, int H, int W, int C, int p, int aug, uint64_t seed,
                         uint32_t step, uint32_t s0, int b_off, __nv_bfloat16* P, cudaStream_t st) {
    vit_patchify_kernel<__nv_bfloat16><<<dim3(B, S), 256, 0, st>>>(x, B, H, W, C, p, aug, make_key(seed), step, s0,
                                                                    b_off, P);
}

// X0[s][b][0] = cls_s + pos_s[0];  X0[s][b][t] = E[s][b][t−1] + pos_s[t]
// one thread per 4 columns of a token row (32-bit index math; D % 4 == 0)
__global__ void vit_embed_kernel(const float* __restrict__ E, const float* __restrict__ cls,
                                 const float* __restrict__ pos, int B, int T, int D, float* __restrict__ X) {
    const int D4 = D >> 2, n4 = B * T * D4, s = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const int row = i / D4, d = (i - row * D4) * 4, b = row / T, t = row - b * T;
    const float4 v = t == 0 ? *reinterpret_cast<const float4*>(cls + (int64_t)s * D + d)
                            : *reinterpret_cast<const float4*>(E + (((int64_t)s * B + b) * (T - 1) + t - 1) * D + d);
    const float4 p = *reinterpret_cast<const float4*>(pos + ((int64_t)s * T + t) * D + d);
    *reinterpret_cast<float4*>(X + ((int64_t)s * B * T + row) * D + d) =
        make_float4(v.x + p.x, v.y + p.y, v.z + p.z, v.w + p.w);
}

void launch_vit_embed(const float* E, const float* cls, const float* pos, int S, int B, int T, int D, float* X,
                      cudaStream_t st) {
    const int n4 = B * T * (D / 4);
    vit_embed_kernel<<<dim3((n4 + 255) / 256, S), 256, 0, st>>>(E, cls, pos, B, T, D, X);
}

// ------------------------------------------------------------------------ LayerNorm
// one warp per row; rows of one sample are `rows` rows `ld` floats apart (ld = D: all tokens;
// ld = T·D: the cls rows); g, b: sampled [s][D]
template <class TY>
__global__ void vit_ln_fwd_kernel(const float* __restrict__ X, int rows, int64_t ld, int64_t sX, int D,
                                  const float* __restrict__ g, const float* __restrict__ bb, TY* __restrict__ Y,
                                  int64_t ldy, int64_t sY, float* __restrict__ stats) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31, s = blockIdx.y;
    if (warp >= rows) return;
    const float* x = X + s * sX + warp * ld;
    float sum = 0.f;
    for (int i = lane; i < D; i += 32) sum += x[i];
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum / D;
    float sq = 0.f;
    for (int i = lane; i < D; i += 32) sq += (x[i] - mean) * (x[i] - mean);
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rstd = rsqrtf(sq / D + 1e-6f);
    TY* y = Y + s * sY + warp * ldy;
    for (int i = lane; i < D; i += 32) stf(y, i, g[(int64_t)s * D + i] * ((x[i] - mean) * rstd) + bb[(int64_t)s * D + i]);
    if (lane == 0) {
        stats[((int64_t)s * rows + warp) * 2] = mean;
        stats[((int64_t)s * rows + warp) * 2 + 1] = rstd;
    }
}

void launch_vit_ln_fwd(const float* X, int S, int rows, int64_t ld, int64_t sX, int D, const float* g, const float* b,
                       float* Y, int64_t ldy, int64_t sY, float* stats, cudaStream_t st) {
    vit_ln_fwd_kernel<float><<<dim3((rows + 7) / 8, S), 256, 0, st>>>(X, rows, ld, sX, D, g, b, Y, ldy, sY, stats);
}
// the same with D = 32·NC known at compile time and RB rows per warp in flight (all loads of a
// warp's rows issued before its reductions: the row-per-warp form waits one memory latency per row)
template <int NC>
__global__ void __launch_bounds__(256) vit_ln_fwd_rows_kernel(const float* __restrict__ X, int rows, int64_t ld,
                                                              int64_t sX, const float* __restrict__ g,
                                                              const float* __restrict__ bb,
                                                              __nv_bfloat16* __restrict__ Y, int64_t ldy, int64_t sY,
                                                              float* __restrict__ stats) {
    constexpr int D = 32 * NC, RB = 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, s = blockIdx.y;
    const int r0 = (blockIdx.x * 8 + warp) * RB;
    float xv[RB][NC];
#pragma unroll
    for (int k = 0; k < RB; ++k)
#pragma unroll
        for (int c = 0; c < NC; ++c) xv[k][c] = r0 + k < rows ? X[s * sX + (r0 + k) * ld + lane + 32 * c] : 0.0f;
    float gl[NC], bl[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        gl[c] = g[(int64_t)s * D + lane + 32 * c];
        bl[c] = bb[(int64_t)s * D + lane + 32 * c];
    }
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        const int r = r0 + k;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < NC; ++c) sum += xv[k][c];
        const float mean = warp_sum(sum) / D;
        float sq = 0.f;
#pragma unroll
        for (int c = 0; c < NC; ++c) sq += (xv[k][c] - mean) * (xv[k][c] - mean);
        const float rstd = rsqrtf(warp_sum(sq) / D + 1e-6f);
        if (r >= rows) continue;
        __nv_bfloat16* y = Y + s * sY + r * ldy;
#pragma unroll
        for (int c = 0; c < NC; ++c) y[lane + 32 * c] = __float2bfloat16_rn(gl[c] * ((xv[k][c] - mean) * rstd) + bl[c]);
        if (lane == 0) {
            stats[((int64_t)s * rows + r) * 2] = mean;
            stats[((int64_t)s * rows + r) * 2 + 1] = rstd;
        }
    }
}

void launch_vit_ln_fwd(const float* X, int S, int rows, int64_t ld, int64_t sX, int D, const float* g, const float* b,
                       __nv_bfloat16* Y, int64_t ldy, int64_t sY, float* stats, cudaStream_t st) {
    const dim3 grid((rows + 31) / 32, S);
#define BNN_LN_FWD(NC)                                                                                          \
    case NC:                                                                                                    \
        vit_ln_fwd_rows_kernel<NC><<<grid, 256, 0, st>>>(X, rows, ld, sX, g, b, Y, ldy, sY, stats);             \
        return;
    if (D % 32 == 0) switch (D / 32) {
            BNN_LN_FWD(1) BNN_LN_FWD(2) BNN_LN_FWD(3) BNN_LN_FWD(4) BNN_LN_FWD(5) BNN_LN_FWD(6) BNN_LN_FWD(7)
            BNN_LN_FWD(8)
            default: break;
        }
#undef BNN_LN_FWD
    vit_ln_fwd_kernel<__nv_bfloat16><<<dim3((rows + 7) / 8, S), 256, 0, st>>>(X, rows, ld, sX, D, g, b, Y, ldy, sY,
                                                                              stats);
}

// dX += rstd·(dx̂ − mean(dx̂) − x̂·mean(dx̂ ⊙ x̂)), dx̂ = dY ⊙ g; dyxh = dY ⊙ x̂ (the g-gradient rows)
template <class TD>
__global__ void vit_ln_bwd_kernel(const TD* __restrict__ dY, int64_t ldy, int64_t sdY, const float* __restrict__ X,
                                  int rows, int64_t ld, int64_t sX, int D, const float* __restrict__ g,
                                  const float* __restrict__ stats, float* __restrict__ dX, float* __restrict__ dyxh) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31, s = blockIdx.y;
    if (warp >= rows) return;
    const float mean = stats[((int64_t)s * rows + warp) * 2], rstd = stats[((int64_t)s * rows + warp) * 2 + 1];
    const float* x = X + s * sX + warp * ld;
    const TD* dy = dY + s * sdY + warp * ldy;
    float m1 = 0.f, m2 = 0.f;
    for (int i = lane; i < D; i += 32) {
        const float xh = (x[i] - mean) * rstd, dxh = ldf(dy, i) * g[(int64_t)s * D + i];
        m1 += dxh;
        m2 += dxh * xh;
    }
    for (int o = 16; o; o >>= 1) {
        m1 += __shfl_xor_sync(0xffffffffu, m1, o);
        m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    m1 /= D;
    m2 /= D;
    float* dx = dX + s * sX + warp * ld;
    float* dg = dyxh + ((int64_t)s * rows + warp) * D;
    for (int i = lane; i < D; i += 32) {
        const float xh = (x[i] - mean) * rstd;
        const float d = ldf(dy, i);
        dx[i] += rstd * (d * g[(int64_t)s * D + i] - m1 - xh * m2);
        dg[i] = d * xh;
    }
}

void launch_vit_ln_bwd(const float* dY, int64_t ldy, int64_t sdY, const float* X, int S, int rows, int64_t ld,
                       int64_t sX, int D, const float* g, const float* stats, float* dX, float* dyxh, cudaStream_t st) {
    vit_ln_bwd_kernel<float><<<dim3((rows + 7) / 8, S), 256, 0, st>>>(dY, ldy, sdY, X, rows, ld, sX, D, g, stats, dX,
                                                                        dyxh);
}
void launch_vit_ln_bwd(const __nv_bfloat16* dY, int64_t ldy, int64_t sdY, const float* X, int S, int rows, int64_t ld,
                       int64_t sX, int D, const float* g, const float* stats, float* dX, float* dyxh, cudaStream_t st) {
    vit_ln_bwd_kernel<__nv_bfloat16><<<dim3((rows + 7) / 8, S), 256, 0, st>>>(dY, ldy, sdY, X, rows, ld, sX, D, g, stats,
                                                                                dX, dyxh);
}

// The same backward over all `rows` token rows of a sample (contiguous, pitch D ≤ 256, D % 32 == 0)
// with the γ / β gradient sources reduced in place: block (q, s) takes rows 64q … 64q + 63 (warp
// w: rows 64q + w + 8k, k = 0…7, in that order), and writes the chunk sums
// part_g[s][q][·] = Σ dY ⊙ x̂ and part_b[s][q][·] = Σ dY (warps added in index order: fixed order,
// deterministic), the inputs of launch_bias_grad — instead of a dY ⊙ x̂ tensor re-read by a
// separate chunk pass. dXb (optional): the bf16 copy of the updated dX rows (the next GEMM operand).
constexpr int kLnMaxC = 8;  // columns per lane (D ≤ 256)
template <int NC>
__global__ void __launch_bounds__(256) vit_ln_bwd_fused_kernel(const float* __restrict__ dY,
                                                               const float* __restrict__ X, int rows,
                                                               const float* __restrict__ g,
                                                               const float* __restrict__ stats,
                                                               float* __restrict__ dX, __nv_bfloat16* __restrict__ dXb,
                                                               float* __restrict__ part_g, float* __restrict__ part_b,
                                                               float* __restrict__ part_x) {
    constexpr int D = 32 * NC, RB = 4;  // RB rows of a warp in flight (all their loads first)
    __shared__ float red[3][8][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = blockIdx.x, s = blockIdx.y;
    const int nq = gridDim.x;
    const int64_t sX = (int64_t)rows * D;
    float gl[NC], ag[NC], ab[NC], ax[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        gl[c] = g[(int64_t)s * D + lane + 32 * c];
        ag[c] = ab[c] = ax[c] = 0.0f;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < 8; k0 += RB) {
        float xv[RB][NC], dv[RB][NC], ov[RB][NC], mean[RB], rstd[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int r = 64 * q + warp + 8 * (k0 + k);
            const bool ok = r < rows;
            const int64_t o = s * sX + (int64_t)r * D + lane;
            mean[k] = ok ? stats[((int64_t)s * rows + r) * 2] : 0.0f;
            rstd[k] = ok ? stats[((int64_t)s * rows + r) * 2 + 1] : 0.0f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                xv[k][c] = ok ? X[o + 32 * c] : 0.0f;
                dv[k][c] = ok ? dY[o + 32 * c] : 0.0f;
                ov[k][c] = ok ? dX[o + 32 * c] : 0.0f;
            }
        }
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int r = 64 * q + warp + 8 * (k0 + k);
            float m1 = 0.f, m2 = 0.f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                xv[k][c] = (xv[k][c] - mean[k]) * rstd[k];
                const float dxh = dv[k][c] * gl[c];
                m1 += dxh;
                m2 += dxh * xv[k][c];
            }
            m1 = warp_sum(m1) * (1.0f / D);
            m2 = warp_sum(m2) * (1.0f / D);
            if (r >= rows) continue;
            const int64_t o = s * sX + (int64_t)r * D + lane;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float v = ov[k][c] + rstd[k] * (dv[k][c] * gl[c] - m1 - xv[k][c] * m2);
                dX[o + 32 * c] = v;
                if (dXb) dXb[o + 32 * c] = __float2bfloat16_rn(v);
                ag[c] += dv[k][c] * xv[k][c];
                ab[c] += dv[k][c];
                ax[c] += v;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        red[0][warp][lane + 32 * c] = ag[c];
        red[1][warp][lane + 32 * c] = ab[c];
        red[2][warp][lane + 32 * c] = ax[c];
    }
    __syncthreads();
    const int nw = part_x ? 3 : 2;
    for (int i = threadIdx.x; i < nw * D; i += blockDim.x) {
        const int w = i / D, n = i - w * D;
        float t = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) t += red[w][j][n];
        (w == 0 ? part_g : w == 1 ? part_b : part_x)[((int64_t)s * nq + q) * D + n] = t;
    }
}

bool vit_ln_bwd_fused_ok(int D) { return D % 32 == 0 && D <= 32 * kLnMaxC; }
void launch_vit_ln_bwd_fused(const float* dY, const float* X, int S, int rows, int D, const float* g,
                             const float* stats, float* dX, __nv_bfloat16* dXb, float* part_g, float* part_b,
                             float* part_x, cudaStream_t st) {
    const dim3 grid((rows + 63) / 64, S);
#define BNN_LN_BWD(NC)                                                                                              \
    case NC:                                                                                                        \
        vit_ln_bwd_fused_kernel<NC><<<grid, 256, 0, st>>>(dY, X, rows, g, stats, dX, dXb, part_g, part_b, part_x); \
        break;
    switch (D / 32) {
        BNN_LN_BWD(1) BNN_LN_BWD(2) BNN_LN_BWD(3) BNN_LN_BWD(4) BNN_LN_BWD(5) BNN_LN_BWD(6) BNN_LN_BWD(7)
        BNN_LN_BWD(8)
        default: break;
    }
#undef BNN_LN_BWD
}

// dUb = bf16(dA ⊙ GELU'(U)) for the BF16 step's fc1 operand, with the fc1 bias source reduced in
// place: part[s][q][·] = Σ over rows 64q … 64q + 63 (in row order) of dA ⊙ GELU'(U) in fp32 —
// the fp32 dU itself is never stored. Block (q, s); thread: 4 adjacent columns (M % 4 == 0).
__global__ void __launch_bounds__(256) vit_gelu_bwd_fused_kernel(const float* __restrict__ U,
                                                                 const float* __restrict__ dA, int rows, int M,
                                                                 __nv_bfloat16* __restrict__ dUb,
                                                                 float* __restrict__ part) {
    const int q = blockIdx.x, s = blockIdx.y, nq = gridDim.x;
    const int r0 = 64 * q, r1 = min(rows, r0 + 64);
    const int64_t base = (int64_t)s * rows * M;
    constexpr int kR = 8;  // rows in flight: all loads of a group before the (branchy) erf work
    for (int c = 4 * threadIdx.x; c < M; c += 4 * blockDim.x) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        for (int rg = r0; rg < r1; rg += kR) {
            float4 u[kR], d[kR];
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                const int64_t i = base + (int64_t)(rg + k) * M + c;
                u[k] = rg + k < r1 ? __ldg(reinterpret_cast<const float4*>(U + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
                d[k] = rg + k < r1 ? __ldg(reinterpret_cast<const float4*>(dA + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                if (rg + k >= r1) break;
                const int64_t i = base + (int64_t)(rg + k) * M + c;
                const float v0 = d[k].x * gelu_df(u[k].x), v1 = d[k].y * gelu_df(u[k].y),
                            v2 = d[k].z * gelu_df(u[k].z), v3 = d[k].w * gelu_df(u[k].w);
                uint2 o;
                o.x = pack_bf16x2(v0, v1);
                o.y = pack_bf16x2(v2, v3);
                *reinterpret_cast<uint2*>(dUb + i) = o;
                a0 += v0, a1 += v1, a2 += v2, a3 += v3;
            }
        }
        *reinterpret_cast<float4*>(part + ((int64_t)s * nq + q) * M + c) = make_float4(a0, a1, a2, a3);
    }
}
void launch_vit_gelu_bwd_fused(const float* U, const float* dA, int S, int rows, int M, __nv_bfloat16* dUb,
                               float* part, cudaStream_t st) {
    vit_gelu_bwd_fused_kernel<<<dim3((rows + 63) / 64, S), 256, 0, st>>>(U, dA, rows, M, dUb, part);
}

// ------------------------------------------------------------------------ attention
// One block per (head h, example b, sample s), 256 threads. Every operand of the head is staged
// in shared memory as a [TP][PP] tile (T ≤ TP rows, zero padded; pitch 68) and each of
// the small products (S = QKᵀ, O = PV; dP = dO Vᵀ, dQ = dS K, dK = dSᵀ Q, dV = Pᵀ dO) is a
// register-tiled SIMT product: a thread owns a 4 × 4 block of the result, reading 4 + 4
// operands per 16 FMAs from shared memory. fp32 throughout (the ViT's parity mode is FP32).
constexpr int kAttT = 68;   // padded token count (T = 65 for 32×32 images, 4×4 patches)
constexpr int kAttP = 68;   // row pitch (floats): 6 tiles = 111 KB, two backward blocks per SM

// C[m][n] (m < Mr, n < Nc, both < kAttT) = Σ_{k<K} A(m, k)·B(k, n), A(m, k) = A[m·am + k·ak],
// B(k, n) = B[k·bk + n·bn]; the 4 × 4 blocks are dealt to the block's threads round-robin and
// handed to `out(m, n, value)`.
template <class F>
__device__ __forceinline__ void att_product(const float* A, int am, int ak, const float* Bm, int bk, int bn, int Mr,
                                            int Nc, int K, F out) {
    const int mt = (Mr + 3) / 4, nt = (Nc + 3) / 4;
    for (int t = threadIdx.x; t < mt * nt; t += blockDim.x) {
        const int m0 = (t / nt) * 4, n0 = (t % nt) * 4;
        float c[4][4] = {};
        for (int k = 0; k < K; ++k) {
            float a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = A[(m0 + i) * am + k * ak];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = Bm[k * bk + (n0 + j) * bn];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) c[i][j] = fmaf(a[i], bb[j], c[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (m0 + i < Mr && n0 + j < Nc) out(m0 + i, n0 + j, c[i][j]);
    }
}

// stage rows [0, T) of `cols` columns (global row pitch ld, column offset c0) into a zero-padded
// [kAttT][kAttP] tile
template <class TI>
__device__ __forceinline__ void att_stage(float* dst, const TI* src, int T, int ld, int c0, int cols) {
    for (int i = threadIdx.x; i < kAttT * kAttP; i += blockDim.x) {
        const int r = i / kAttP, e = i - r * kAttP;
        dst[i] = (r < T && e < cols) ? ldf(src, (int64_t)r * ld + c0 + e) : 0.0f;
    }
}

// transposed: dst[e][r] = src[r][c0 + e] (so that a product reading the operand along its rows
// walks consecutive shared addresses across the warp — a column walk at pitch 72 hits one bank)
template <class TI>
__device__ __forceinline__ void att_stage_t(float* dst, const TI* src, int T, int ld, int c0, int cols) {
    for (int i = threadIdx.x; i < kAttT * kAttP; i += blockDim.x) {
        const int e = i / kAttP, r = i - e * kAttP;
        dst[i] = (r < T && e < cols) ? ldf(src, (int64_t)r * ld + c0 + e) : 0.0f;
    }
}

template <class TO>
__global__ void __launch_bounds__(256) vit_attn_fwd_kernel(const float* __restrict__ QKV, int B, int T, int D, int dh,
                                                           TO* __restrict__ O, float* __restrict__ A) {
    extern __shared__ float sm[];
    const int h = blockIdx.x, b = blockIdx.y, s = blockIdx.z, nh = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    float* Qs = sm;
    float* Ks = Qs + kAttT * kAttP;
    float* Vs = Ks + kAttT * kAttP;
    float* Ps = Vs + kAttT * kAttP;
    const float* base = QKV + ((int64_t)s * B + b) * T * 3 * D;
    att_stage(Qs, base, T, 3 * D, h * dh, dh);
    att_stage_t(Ks, base, T, 3 * D, D + h * dh, dh);  // Kᵀ
    att_stage(Vs, base, T, 3 * D, 2 * D + h * dh, dh);
    __syncthreads();
    const float sc = rsqrtf((float)dh);
    // S = Q Kᵀ / √dh
    att_product(Qs, kAttP, 1, Ks, kAttP, 1, T, T, dh, [&](int m, int n, float v) { Ps[m * kAttP + n] = v * sc; });
    __syncthreads();
    float* arow_base = A + (((int64_t)s * B + b) * nh + h) * T * T;
    for (int i = warp; i < T; i += nw) {  // row softmax, kept for the backward
        float* pr = Ps + i * kAttP;
        float mx = -INFINITY;
        for (int j = lane; j < T; j += 32) mx = fmaxf(mx, pr[j]);
        mx = warp_max(mx);
        float se = 0.f;
        for (int j = lane; j < T; j += 32) {
            const float e = __expf(pr[j] - mx);
            pr[j] = e;
            se += e;
        }
        se = warp_sum(se);
        const float inv = 1.0f / se;
        for (int j = lane; j < T; j += 32) {
            pr[j] *= inv;
            arow_base[(int64_t)i * T + j] = pr[j];
        }
    }
    __syncthreads();
    // O = P V
    TO* ob = O + ((int64_t)s * B + b) * T * D + h * dh;
    att_product(Ps, kAttP, 1, Vs, kAttP, 1, T, dh, T, [&](int m, int n, float v) { stf(ob, (int64_t)m * D + n, v); });
}

template <class TO>
static void attn_fwd_t(const float* QKV, int S, int B, int T, int D, int heads, TO* O, float* A, cudaStream_t st) {
    const size_t smem = sizeof(float) * 4 * kAttT * kAttP;
    ensure_smem_attr(reinterpret_cast<const void*>(vit_attn_fwd_kernel<TO>), (int)smem);
    vit_attn_fwd_kernel<TO><<<dim3(heads, B, S), 256, smem, st>>>(QKV, B, T, D, D / heads, O, A);
}
bool attn_tc_ok(int T, int dh);
template <class TO>
static void attn_fwd_tc(const float*, int, int, int, int, int, TO*, float*, cudaStream_t);
template <class TD>
static void attn_bwd_tc(const float*, const float*, const TD*, int, int, int, int, int, float*, cudaStream_t);

void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, float* O, float* A,
                         cudaStream_t st) {
    attn_fwd_t(QKV, S, B, T, D, heads, O, A, st);
}
void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, __nv_bfloat16* O, float* A,
                         cudaStream_t st) {
    if (attn_tc_ok(T, D / heads))
        attn_fwd_tc(QKV, S, B, T, D, heads, O, A, st);
    else
        attn_fwd_t(QKV, S, B, T, D, heads, O, A, st);
}

// dP = dO Vᵀ; dS = A ⊙ (dP − rowsum(A ⊙ dP)) / √dh; dQ = dS K; dK = dSᵀ Q; dV = Aᵀ dO —
// written into dQKV (Q | K | V columns of head h)
template <class TD>
__global__ void __launch_bounds__(256) vit_attn_bwd_kernel(const float* __restrict__ QKV, const float* __restrict__ A,
                                                           const TD* __restrict__ dO, int B, int T, int D, int dh,
                                                           float* __restrict__ dQKV) {
    extern __shared__ float sm[];
    const int h = blockIdx.x, b = blockIdx.y, s = blockIdx.z, nh = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr int TILE = kAttT * kAttP;
    float *Qs = sm, *Ks = sm + TILE, *Vs = sm + 2 * TILE, *dOs = sm + 3 * TILE, *As = sm + 4 * TILE, *dSs = sm + 5 * TILE;
    const float* base = QKV + ((int64_t)s * B + b) * T * 3 * D;
    att_stage(Qs, base, T, 3 * D, h * dh, dh);
    att_stage(Ks, base, T, 3 * D, D + h * dh, dh);
    att_stage_t(Vs, base, T, 3 * D, 2 * D + h * dh, dh);  // Vᵀ
    att_stage(dOs, dO + ((int64_t)s * B + b) * T * D, T, D, h * dh, dh);
    att_stage(As, A + (((int64_t)s * B + b) * nh + h) * T * T, T, T, 0, T);
    __syncthreads();
    att_product(dOs, kAttP, 1, Vs, kAttP, 1, T, T, dh, [&](int m, int n, float v) { dSs[m * kAttP + n] = v; });
    __syncthreads();
    const float sc = rsqrtf((float)dh);
    for (int i = warp; i < T; i += nw) {
        float rd = 0.f;
        for (int j = lane; j < T; j += 32) rd += As[i * kAttP + j] * dSs[i * kAttP + j];
        rd = warp_sum(rd);
        for (int j = lane; j < T; j += 32) dSs[i * kAttP + j] = As[i * kAttP + j] * (dSs[i * kAttP + j] - rd) * sc;
    }
    __syncthreads();
    float* out = dQKV + ((int64_t)s * B + b) * T * 3 * D;
    att_product(dSs, kAttP, 1, Ks, kAttP, 1, T, dh, T,
                [&](int m, int n, float v) { out[(int64_t)m * 3 * D + h * dh + n] = v; });
    att_product(dSs, 1, kAttP, Qs, kAttP, 1, T, dh, T,
                [&](int m, int n, float v) { out[(int64_t)m * 3 * D + D + h * dh + n] = v; });
    att_product(As, 1, kAttP, dOs, kAttP, 1, T, dh, T,
                [&](int m, int n, float v) { out[(int64_t)m * 3 * D + 2 * D + h * dh + n] = v; });
}

template <class TD>
static void attn_bwd_t(const float* QKV, const float* A, const TD* dO, int S, int B, int T, int D, int heads,
                       float* dQKV, cudaStream_t st) {
    const size_t smem = sizeof(float) * 6 * kAttT * kAttP;
    ensure_smem_attr(reinterpret_cast<const void*>(vit_attn_bwd_kernel<TD>), (int)smem);
    vit_attn_bwd_kernel<TD><<<dim3(heads, B, S), 256, smem, st>>>(QKV, A, dO, B, T, D, D / heads, dQKV);
}
void launch_vit_attn_bwd(const float* QKV, const float* A, const float* dO, int S, int B, int T, int D, int heads,
                         float* dQKV, cudaStream_t st) {
    attn_bwd_t(QKV, A, dO, S, B, T, D, heads, dQKV, st);
}
void launch_vit_attn_bwd_tf32(const float* QKV, const float* A, const float* dO, int S, int B, int T, int D,
                              int heads, float* dQKV, cudaStream_t st) {
    if (attn_tc_ok(T, D / heads))
        attn_bwd_tc(QKV, A, dO, S, B, T, D, heads, dQKV, st);
    else
        attn_bwd_t(QKV, A, dO, S, B, T, D, heads, dQKV, st);
}
void launch_vit_attn_bwd(const float* QKV, const float* A, const __nv_bfloat16* dO, int S, int B, int T, int D,
                         int heads, float* dQKV, cudaStream_t st) {
    if (attn_tc_ok(T, D / heads))
        attn_bwd_tc(QKV, A, dO, S, B, T, D, heads, dQKV, st);
    else
        attn_bwd_t(QKV, A, dO, S, B, T, D, heads, dQKV, st);
}

// ------------------------------------------------------------------------ attention, tensor cores
// The BF16 step's attention (the FP32 parity mode keeps the SIMT kernels above): the same block
// per (h, b, s), with each small product on the warp-level tensor-core MMA
// mma.sync.m16n8k8 in TF32 (fp32 accumulate). Operands are staged once as natural [token][e]
// tiles of 72 rows (T ≤ 72, zero rows T..71 so every padded reduction index multiplies zeros),
// pre-rounded to TF32 (cvt.rna); a product reads a tile as A(m, k) = X[m·am + k·ak] so a
// transposed operand needs no second copy. The pitch decides the bank pattern of the fragment
// loads: ≡ 4 or 12 (mod 32) makes the row walk (am = pitch) conflict-free, ≡ 8 the column walk.
// m-tiles run over 80 rows: rows 72..79 read the next tile (finite values) and their results are
// dropped. TF32 (10-bit mantissa) is finer than the BF16 operands of the surrounding projections.
constexpr int kTcRows = 72;               // token rows per tile (9 k-steps of 8)
constexpr int kTcSlack = 8 * 80;          // floats after the last tile (pitch ≤ 80) for the 80-row m-tiles

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// C(m, n) = Σ_{k < 8·Kt} A(m, k)·B(k, n) over m < 16·Mt, n < 8·Nt; A(m, k) = A[m·am + k·ak],
// B(k, n) = B[k·bk + n·bn] (TF32 bit patterns, or fp32 rounded on load when CVT_A). A warp owns
// 16 × 16 blocks (two n8 tiles sharing the A fragment); at most kHold blocks per warp are kept
// and handed to out(m, n, v) — for every m, n — after the whole product (after a block barrier
// when SYNC, so the output may overwrite an operand). Fragment layout of m16n8k8 (PTX ISA):
// g = lane/4, q = lane%4; a = (g, q), (g+8, q), (g, q+4), (g+8, q+4); b = (q, g), (q+4, g);
// c = (g, 2q), (g, 2q+1), (g+8, 2q), (g+8, 2q+1).
template <bool CVT_A, bool SYNC, int kHold, class F>
__device__ __forceinline__ void att_mma(const uint32_t* A, int am, int ak, const uint32_t* Bm, int bk, int bn, int Mt,
                                        int Nt, int Kt, F out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int nt2 = (Nt + 1) >> 1, tiles = Mt * nt2;
    float c[kHold][2][4];
#pragma unroll
    for (int h = 0; h < kHold; ++h)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) c[h][u][v] = 0.0f;
#pragma unroll
    for (int h = 0; h < kHold; ++h) {
        const int w = warp + h * nw;
        if (w < tiles) {
            const int m0 = (w / nt2) * 16, n0 = (w % nt2) * 16;
            const bool two = n0 + 8 < Nt * 8;
            const uint32_t* a0p = A + (m0 + g) * am + q * ak;
            const uint32_t* b0p = Bm + q * bk + (n0 + g) * bn;
            for (int k0 = 0; k0 < Kt * 8; k0 += 8) {
                const uint32_t* ap = a0p + k0 * ak;
                uint32_t a[4] = {ap[0], ap[8 * am], ap[4 * ak], ap[8 * am + 4 * ak]};
                if (CVT_A) {
#pragma unroll
                    for (int v = 0; v < 4; ++v) a[v] = to_tf32(__uint_as_float(a[v]));
                }
                const uint32_t* bp = b0p + k0 * bk;
                mma_tf32(c[h][0], a, bp[0], bp[4 * bk]);
                if (two) mma_tf32(c[h][1], a, bp[8 * bn], bp[4 * bk + 8 * bn]);
            }
        }
    }
    if (SYNC) __syncthreads();
#pragma unroll
    for (int h = 0; h < kHold; ++h) {
        const int w = warp + h * nw;
        if (w < tiles) {
            const int m0 = (w / nt2) * 16, n0 = (w % nt2) * 16;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int n = n0 + 8 * u + 2 * q;
                if (n < Nt * 8) {
                    out(m0 + g, n, c[h][u][0]);
                    out(m0 + g, n + 1, c[h][u][1]);
                    out(m0 + g + 8, n, c[h][u][2]);
                    out(m0 + g + 8, n + 1, c[h][u][3]);
                }
            }
        }
    }
}

// dst[r][e] = tf32(src[r·ld + c0 + e]) for r < T, e < cols (cols % 4 == 0), zero rows T..71
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
__device__ __forceinline__ void ld4(const __nv_bfloat16* p, float (&v)[4]) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.x));
    const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.y));
    v[0] = lo.x, v[1] = lo.y, v[2] = hi.x, v[3] = hi.y;
}
// Staging is latency-bound (one block's tiles are ~50 KB read once): every thread issues all of
// its global loads before the first shared store, so a block waits about one memory latency per
// staging phase rather than one per loop trip.
constexpr int kStageIt = 5;  // ⌈72 rows · 16 float4 / 256 threads⌉ (dh ≤ 64)

// NT tiles dst[t][r][e] = tf32(src[r·ld + c0[t] + e]) for r < T, e < cols (cols % 4 == 0; zero
// rows T..71), from one row-major source
template <int NT, int IT = kStageIt, class TI>
__device__ __forceinline__ void tc_stage(uint32_t* const (&dst)[NT], const int (&pitch)[NT], const TI* src, int T,
                                         int64_t ld, const int (&c0)[NT], int cols) {
    const int c4 = cols >> 2, total = kTcRows * c4;
    float v[IT][NT][4];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        const int i = threadIdx.x + u * blockDim.x, r = i / c4, e = (i - r * c4) * 4;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (i < total && r < T) {
                ld4(src + (int64_t)r * ld + c0[t] + e, v[u][t]);
            } else {
                v[u][t][0] = v[u][t][1] = v[u][t][2] = v[u][t][3] = 0.0f;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        const int i = threadIdx.x + u * blockDim.x, r = i / c4, e = (i - r * c4) * 4;
        if (i < total) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                uint4 o;
                o.x = to_tf32(v[u][t][0]), o.y = to_tf32(v[u][t][1]), o.z = to_tf32(v[u][t][2]),
                o.w = to_tf32(v[u][t][3]);
                *reinterpret_cast<uint4*>(dst[t] + r * pitch[t] + e) = o;
            }
        }
    }
}


// Forward, one warp per 16 query rows (FlashAttention-2-style, the whole row in registers): the
// block (5 warps, rows 16w..16w+15) stages K and V once; each warp loads its Q fragments straight from global
// memory, forms S = Q Kᵀ for all 72 key columns (9 accumulator tiles), takes the row softmax
// inside its quads (a row's 72 values live in the 4 lanes of one quad), writes A, and feeds P to
// P·V as the A operand after moving it from the accumulator layout (g, 2q | 2q+1) to the operand
// layout (g, q | q+4) with quad shuffles. No block barrier after staging; 40 KB of shared memory.
constexpr int kFk = 68, kFv = 72;  // K: row walk (B(k = e, n = j) = K[j][e]); V: column walk
template <int KD, class TO>
__global__ void __launch_bounds__(160) vit_attn_fwd_tc_kernel(const float* __restrict__ QKV, int B, int T, int D,
                                                              TO* __restrict__ O, float* __restrict__ A) {
    constexpr int dh = 8 * KD, NT = kTcRows / 8;
    extern __shared__ __align__(16) uint32_t smu[];
    const int h = blockIdx.x, b = blockIdx.y, s = blockIdx.z, nh = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    uint32_t* Ks = smu;
    uint32_t* Vs = Ks + kTcRows * kFk;
    const float* base = QKV + ((int64_t)s * B + b) * T * 3 * D;
    {
        uint32_t* const dst[2] = {Ks, Vs};
        const int pitch[2] = {kFk, kFv}, c0[2] = {D + h * dh, 2 * D + h * dh};
        tc_stage<2, 8>(dst, pitch, base, T, 3 * D, c0, dh);
    }
    const int m0 = 16 * warp, r0 = m0 + g, r1 = r0 + 8;
    uint32_t qa[KD][4];  // Q rows r0, r1 as m16n8k8 A fragments
#pragma unroll
    for (int k = 0; k < KD; ++k) {
        const float* q0 = base + (int64_t)r0 * 3 * D + h * dh + 8 * k + q;
        const float* q1 = base + (int64_t)r1 * 3 * D + h * dh + 8 * k + q;
        qa[k][0] = to_tf32(r0 < T ? __ldg(q0) : 0.0f);
        qa[k][1] = to_tf32(r1 < T ? __ldg(q1) : 0.0f);
        qa[k][2] = to_tf32(r0 < T ? __ldg(q0 + 4) : 0.0f);
        qa[k][3] = to_tf32(r1 < T ? __ldg(q1 + 4) : 0.0f);
    }
    __syncthreads();
    if (m0 >= T) return;  // 5 warps cover T ≤ 72 rows (the staging needs all 160 threads)
    float sa[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        sa[n][0] = sa[n][1] = sa[n][2] = sa[n][3] = 0.0f;
        const uint32_t* kp = Ks + (8 * n + g) * kFk + q;
#pragma unroll
        for (int k = 0; k < KD; ++k) mma_tf32(sa[n], qa[k], kp[8 * k], kp[8 * k + 4]);
    }
    // row softmax of S / √dh over the columns < T; rows r0 (elements 0, 1) and r1 (2, 3)
    const float sc = rsqrtf((float)dh) * 1.4426950408889634f;  // exp(x) = 2^(x·log2 e)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const bool ok = 8 * n + 2 * q + u < T;
            sa[n][u] = ok ? sa[n][u] * sc : -INFINITY;
            sa[n][2 + u] = ok ? sa[n][2 + u] * sc : -INFINITY;
            mx0 = fmaxf(mx0, sa[n][u]);
            mx1 = fmaxf(mx1, sa[n][2 + u]);
        }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    float se0 = 0.0f, se1 = 0.0f;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            sa[n][u] = exp2f(sa[n][u] - mx0);
            sa[n][2 + u] = exp2f(sa[n][2 + u] - mx1);
            se0 += sa[n][u];
            se1 += sa[n][2 + u];
        }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        se0 += __shfl_xor_sync(0xffffffffu, se0, o);
        se1 += __shfl_xor_sync(0xffffffffu, se1, o);
    }
    const float inv0 = 1.0f / se0, inv1 = 1.0f / se1;
    float* ab = A + (((int64_t)s * B + b) * nh + h) * T * T;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = 8 * n + 2 * q + u;
            sa[n][u] *= inv0;
            sa[n][2 + u] *= inv1;
            if (j < T) {
                if (r0 < T) ab[(int64_t)r0 * T + j] = sa[n][u];
                if (r1 < T) ab[(int64_t)r1 * T + j] = sa[n][2 + u];
            }
        }
    // O = P V: the A fragment of k-step kk is columns 8kk + q (+4) of rows r0, r1, held by quad
    // lanes q/2 and 2 + q/2 as element q % 2
    float oa[KD][4];
#pragma unroll
    for (int n = 0; n < KD; ++n) oa[n][0] = oa[n][1] = oa[n][2] = oa[n][3] = 0.0f;
    const int srcA = (lane & ~3) | (q >> 1), srcB = srcA + 2;
    const bool odd = q & 1;
#pragma unroll
    for (int kk = 0; kk < NT; ++kk) {
        float x[4][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            x[0][u] = __shfl_sync(0xffffffffu, sa[kk][u], srcA);
            x[1][u] = __shfl_sync(0xffffffffu, sa[kk][2 + u], srcA);
            x[2][u] = __shfl_sync(0xffffffffu, sa[kk][u], srcB);
            x[3][u] = __shfl_sync(0xffffffffu, sa[kk][2 + u], srcB);
        }
        const uint32_t pa[4] = {to_tf32(odd ? x[0][1] : x[0][0]), to_tf32(odd ? x[1][1] : x[1][0]),
                                to_tf32(odd ? x[2][1] : x[2][0]), to_tf32(odd ? x[3][1] : x[3][0])};
        const uint32_t* vp = Vs + (8 * kk + q) * kFv + g;
#pragma unroll
        for (int n = 0; n < KD; ++n) mma_tf32(oa[n], pa, vp[8 * n], vp[4 * kFv + 8 * n]);
    }
    TO* ob = O + ((int64_t)s * B + b) * T * D + h * dh;
#pragma unroll
    for (int n = 0; n < KD; ++n) {
        const int e = 8 * n + 2 * q;
        if (r0 < T) {
            stf(ob, (int64_t)r0 * D + e, oa[n][0]);
            stf(ob, (int64_t)r0 * D + e + 1, oa[n][1]);
        }
        if (r1 < T) {
            stf(ob, (int64_t)r1 * D + e, oa[n][2]);
            stf(ob, (int64_t)r1 * D + e + 1, oa[n][3]);
        }
    }
}

bool attn_tc_ok(int T, int dh) { return T >= 1 && T <= kTcRows && (dh == 16 || dh == 32 || dh == 64); }

template <int KD, class TO>
static void attn_fwd_tc_kd(const float* QKV, int S, int B, int T, int D, int heads, TO* O, float* A,
                           cudaStream_t st) {
    const size_t smem = sizeof(uint32_t) * kTcRows * (kFk + kFv);
    ensure_smem_attr(reinterpret_cast<const void*>(vit_attn_fwd_tc_kernel<KD, TO>), (int)smem);
    vit_attn_fwd_tc_kernel<KD, TO><<<dim3(heads, B, S), 160, smem, st>>>(QKV, B, T, D, O, A);
}
template <class TO>
static void attn_fwd_tc(const float* QKV, int S, int B, int T, int D, int heads, TO* O, float* A, cudaStream_t st) {
    switch (D / heads) {
        case 16: attn_fwd_tc_kd<2>(QKV, S, B, T, D, heads, O, A, st); break;
        case 32: attn_fwd_tc_kd<4>(QKV, S, B, T, D, heads, O, A, st); break;
        default: attn_fwd_tc_kd<8>(QKV, S, B, T, D, heads, O, A, st); break;
    }
}

// Backward, the same warp per 16 query rows i: dP = dO Vᵀ, the row sums Σ_j P ⊙ dP and
// dS = P ⊙ (dP − rowsum) / √dh stay in registers (P read in the accumulator layout straight from
// A), and dQ = dS K is formed per warp (dS moved to the operand layout by quad shuffles). dK = dSᵀ Q
// and dV = Pᵀ dO reduce over i — across the warps — so dS and P are then written into the slots
// of V and K and both products run block-wide (att_mma, column-walk operands).
constexpr int kBp = 72;  // every backward tile: K, Q, dO, P are column-walked; V / dS share 72
template <int KD, class TD>
__global__ void __launch_bounds__(160, 2) vit_attn_bwd_tc_kernel(const float* __restrict__ QKV,
                                                              const float* __restrict__ A,
                                                              const TD* __restrict__ dO, int B, int T, int D,
                                                              float* __restrict__ dQKV) {
    constexpr int dh = 8 * KD, NT = kTcRows / 8;
    extern __shared__ __align__(16) uint32_t smu[];
    const int h = blockIdx.x, b = blockIdx.y, s = blockIdx.z, nh = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    constexpr int TILE = kTcRows * kBp;
    uint32_t* Ks = smu;            // later P
    uint32_t* Vs = smu + TILE;     // later dS
    uint32_t* Qs = smu + 2 * TILE;
    uint32_t* dOs = smu + 3 * TILE;
    const float* base = QKV + ((int64_t)s * B + b) * T * 3 * D;
    const TD* dOb = dO + ((int64_t)s * B + b) * T * D + h * dh;
    {
        uint32_t* const dst[3] = {Ks, Vs, Qs};
        const int pitch[3] = {kBp, kBp, kBp}, c0[3] = {D + h * dh, 2 * D + h * dh, h * dh};
        tc_stage<3, 8>(dst, pitch, base, T, 3 * D, c0, dh);
        uint32_t* const dst1[1] = {dOs};
        const int pitch1[1] = {kBp}, c01[1] = {0};
        tc_stage<1, 8>(dst1, pitch1, dOb, T, D, c01, dh);
    }
    const int m0 = 16 * warp, r0 = m0 + g, r1 = r0 + 8;
    const bool active = m0 < T;
    float* out = dQKV + ((int64_t)s * B + b) * T * 3 * D + h * dh;
    float pr[NT][4] = {}, ds[NT][4] = {};
    if (active) {  // P rows r0, r1 in the accumulator layout, straight from A
        const float* ab = A + (((int64_t)s * B + b) * nh + h) * T * T;
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = 8 * n + 2 * q + u;
                pr[n][u] = (r0 < T && j < T) ? __ldg(ab + (int64_t)r0 * T + j) : 0.0f;
                pr[n][2 + u] = (r1 < T && j < T) ? __ldg(ab + (int64_t)r1 * T + j) : 0.0f;
            }
    }
    __syncthreads();
    if (active) {
        // dP = dO Vᵀ: A = the staged dO rows, B(k = e, n = j) = V[j][e]
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            ds[n][0] = ds[n][1] = ds[n][2] = ds[n][3] = 0.0f;
            const uint32_t* vp = Vs + (8 * n + g) * kBp + q;
#pragma unroll
            for (int k = 0; k < KD; ++k) {
                const uint32_t* ap = dOs + r0 * kBp + 8 * k + q;
                const uint32_t af[4] = {ap[0], ap[8 * kBp], ap[4], ap[8 * kBp + 4]};
                mma_tf32(ds[n], af, vp[8 * k], vp[8 * k + 4]);
            }
        }
        float rd0 = 0.0f, rd1 = 0.0f;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            rd0 += pr[n][0] * ds[n][0] + pr[n][1] * ds[n][1];
            rd1 += pr[n][2] * ds[n][2] + pr[n][3] * ds[n][3];
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            rd0 += __shfl_xor_sync(0xffffffffu, rd0, o);
            rd1 += __shfl_xor_sync(0xffffffffu, rd1, o);
        }
        const float sc = rsqrtf((float)dh);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            ds[n][0] = pr[n][0] * (ds[n][0] - rd0) * sc;
            ds[n][1] = pr[n][1] * (ds[n][1] - rd0) * sc;
            ds[n][2] = pr[n][2] * (ds[n][2] - rd1) * sc;
            ds[n][3] = pr[n][3] * (ds[n][3] - rd1) * sc;
        }
        // dQ = dS K: A fragment of k-step kk from quad lanes q/2, 2 + q/2; B(k = j, n = e) = K[j][e]
        float qa[KD][4];
#pragma unroll
        for (int n = 0; n < KD; ++n) qa[n][0] = qa[n][1] = qa[n][2] = qa[n][3] = 0.0f;
        const int srcA = (lane & ~3) | (q >> 1), srcB = srcA + 2;
        const bool odd = q & 1;
#pragma unroll
        for (int kk = 0; kk < NT; ++kk) {
            float x[4][2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                x[0][u] = __shfl_sync(0xffffffffu, ds[kk][u], srcA);
                x[1][u] = __shfl_sync(0xffffffffu, ds[kk][2 + u], srcA);
                x[2][u] = __shfl_sync(0xffffffffu, ds[kk][u], srcB);
                x[3][u] = __shfl_sync(0xffffffffu, ds[kk][2 + u], srcB);
            }
            const uint32_t af[4] = {to_tf32(odd ? x[0][1] : x[0][0]), to_tf32(odd ? x[1][1] : x[1][0]),
                                    to_tf32(odd ? x[2][1] : x[2][0]), to_tf32(odd ? x[3][1] : x[3][0])};
            const uint32_t* kp = Ks + (8 * kk + q) * kBp + g;
#pragma unroll
            for (int n = 0; n < KD; ++n) mma_tf32(qa[n], af, kp[8 * n], kp[4 * kBp + 8 * n]);
        }
#pragma unroll
        for (int n = 0; n < KD; ++n) {
            const int e = 8 * n + 2 * q;
            if (r0 < T) *reinterpret_cast<float2*>(out + (int64_t)r0 * 3 * D + e) = make_float2(qa[n][0], qa[n][1]);
            if (r1 < T) *reinterpret_cast<float2*>(out + (int64_t)r1 * 3 * D + e) = make_float2(qa[n][2], qa[n][3]);
        }
    }
    __syncthreads();  // V and K are consumed: their slots take dS and P (rows ≥ T zero)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = 8 * n + 2 * q + u;
            if (r0 < kTcRows) {
                Vs[r0 * kBp + j] = active ? to_tf32(ds[n][u]) : 0u;
                Ks[r0 * kBp + j] = active ? to_tf32(pr[n][u]) : 0u;
            }
            if (r1 < kTcRows) {
                Vs[r1 * kBp + j] = active ? to_tf32(ds[n][2 + u]) : 0u;
                Ks[r1 * kBp + j] = active ? to_tf32(pr[n][2 + u]) : 0u;
            }
        }
    __syncthreads();
    const int Mt = (T + 15) >> 4, Kt = kTcRows / 8;
    // dK = dSᵀ Q: A(m = j, k = i) = dS[i][j], B(k = i, n = e) = Q[i][e]
    att_mma<false, false, 4>(Vs, 1, kBp, Qs, kBp, 1, Mt, KD, Kt, [&](int m, int n, float v) {
        if (m < T) out[(int64_t)m * 3 * D + D + n] = v;
    });
    // dV = Pᵀ dO: A(m = j, k = i) = P[i][j], B(k = i, n = e) = dO[i][e]
    att_mma<false, false, 4>(Ks, 1, kBp, dOs, kBp, 1, Mt, KD, Kt, [&](int m, int n, float v) {
        if (m < T) out[(int64_t)m * 3 * D + 2 * D + n] = v;
    });
}

template <int KD, class TD>
static void attn_bwd_tc_kd(const float* QKV, const float* A, const TD* dO, int S, int B, int T, int D, int heads,
                           float* dQKV, cudaStream_t st) {
    const size_t smem = sizeof(uint32_t) * (4 * kTcRows * kBp + kTcSlack);
    ensure_smem_attr(reinterpret_cast<const void*>(vit_attn_bwd_tc_kernel<KD, TD>), (int)smem);
    vit_attn_bwd_tc_kernel<KD, TD><<<dim3(heads, B, S), 160, smem, st>>>(QKV, A, dO, B, T, D, dQKV);
}
template <class TD>
static void attn_bwd_tc(const float* QKV, const float* A, const TD* dO, int S, int B, int T, int D, int heads,
                        float* dQKV, cudaStream_t st) {
    switch (D / heads) {
        case 16: attn_bwd_tc_kd<2>(QKV, A, dO, S, B, T, D, heads, dQKV, st); break;
        case 32: attn_bwd_tc_kd<4>(QKV, A, dO, S, B, T, D, heads, dQKV, st); break;
        default: attn_bwd_tc_kd<8>(QKV, A, dO, S, B, T, D, heads, dQKV, st); break;
    }
}

// ------------------------------------------------------------------------ elementwise

__global__ void vit_gelu_kernel(const float* __restrict__ U, int64_t n, float* __restrict__ Aout) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        Aout[i] = gelu_f(U[i]);
}
__global__ void vit_gelu_bwd_kernel(const float* __restrict__ U, int64_t n, float* __restrict__ dA) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dA[i] *= gelu_df(U[i]);
}
__global__ void vit_add_kernel(float* __restrict__ Y, const float* __restrict__ X, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        Y[i] += X[i];
}
// rows r of [S][rows][D] that are token t0 + (r mod per)… : out[s][b][k][d] = in[s][b][t0 + k][d]
__global__ void vit_gather_tokens_kernel(const float* __restrict__ in, int B, int T, int t0, int nt, int D,
                                         float* __restrict__ out) {
    const int D4 = D >> 2, n4 = B * nt * D4, s = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const int row = i / D4, d = (i - row * D4) * 4, b = row / nt, k = row - b * nt;
    *reinterpret_cast<float4*>(out + ((int64_t)s * B * nt + row) * D + d) =
        *reinterpret_cast<const float4*>(in + (((int64_t)s * B + b) * T + t0 + k) * D + d);
}

// fp32 → bf16 maps, 4 elements per thread and trip (16-B loads, 8-B stores; n % 4 == 0 and
// aligned buffers, see vec4_ok), two trips' loads in flight
template <bool GELU>
__global__ void vit_to_bf16x4_kernel(const float* __restrict__ x, int64_t n4, __nv_bfloat16* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 2 * stride) {
        const bool two = i + stride < n4;
        const float4 a = __ldg(reinterpret_cast<const float4*>(x) + i);
        const float4 b = two ? __ldg(reinterpret_cast<const float4*>(x) + i + stride) : a;
        auto f = [](float v) { return GELU ? gelu_f(v) : v; };
        reinterpret_cast<uint2*>(y)[i] = make_uint2(pack_bf16x2(f(a.x), f(a.y)), pack_bf16x2(f(a.z), f(a.w)));
        if (two)
            reinterpret_cast<uint2*>(y)[i + stride] =
                make_uint2(pack_bf16x2(f(b.x), f(b.y)), pack_bf16x2(f(b.z), f(b.w)));
    }
}
static bool vec4_ok(const void* a, const void* b, int64_t n) {
    return n % 4 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 7) == 0;
}
__global__ void vit_gelu_bf16_kernel(const float* __restrict__ U, int64_t n, __nv_bfloat16* __restrict__ Aout) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        Aout[i] = __float2bfloat16_rn(gelu_f(U[i]));
}
// dU = dA ⊙ GELU'(U) from the bf16 dgrad output: fp32 (bias gradient) and bf16 (next GEMM operand)
__global__ void vit_gelu_bwd_bf16_kernel(const float* __restrict__ U, int64_t n, const __nv_bfloat16* __restrict__ dA,
                                         float* __restrict__ dU, __nv_bfloat16* __restrict__ dUb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = __bfloat162float(dA[i]) * gelu_df(U[i]);
        dU[i] = v;
        dUb[i] = __float2bfloat16_rn(v);
    }
}
__global__ void vit_cast_bf16_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}
void launch_vit_gelu(const float* U, int64_t n, __nv_bfloat16* A, cudaStream_t st) {
    if (vec4_ok(U, A, n)) {
        vit_to_bf16x4_kernel<true><<<(int)std::min<int64_t>((n / 4 + 511) / 512, 148 * 8), 256, 0, st>>>(U, n / 4, A);
        return;
    }
    vit_gelu_bf16_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(U, n, A);
}
void launch_vit_gelu_bwd(const float* U, int64_t n, const __nv_bfloat16* dA, float* dU, __nv_bfloat16* dUb,
                         cudaStream_t st) {
    vit_gelu_bwd_bf16_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(U, n, dA, dU, dUb);
}
__global__ void vit_widen_kernel(const __nv_bfloat16* __restrict__ x, int64_t n, float* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __bfloat162float(x[i]);
}
void launch_vit_widen(const __nv_bfloat16* x, int64_t n, float* y, cudaStream_t st) {
    vit_widen_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(x, n, y);
}
__global__ void vit_gelu_bwd_cast_kernel(const float* __restrict__ U, int64_t n, float* __restrict__ dA,
                                         __nv_bfloat16* __restrict__ dUb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = dA[i] * gelu_df(U[i]);
        dA[i] = v;
        dUb[i] = __float2bfloat16_rn(v);
    }
}
void launch_vit_gelu_bwd_cast(const float* U, int64_t n, float* dA, __nv_bfloat16* dUb, cudaStream_t st) {
    vit_gelu_bwd_cast_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(U, n, dA, dUb);
}
void launch_vit_cast_bf16(const float* x, int64_t n, __nv_bfloat16* y, cudaStream_t st) {
    if (vec4_ok(x, y, n)) {
        vit_to_bf16x4_kernel<false><<<(int)std::min<int64_t>((n / 4 + 511) / 512, 148 * 8), 256, 0, st>>>(x, n / 4, y);
        return;
    }
    vit_cast_bf16_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(x, n, y);
}
void launch_vit_gelu(const float* U, int64_t n, float* A, cudaStream_t st) {
    vit_gelu_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(U, n, A);
}
void launch_vit_gelu_bwd(const float* U, int64_t n, float* dA, cudaStream_t st) {
    vit_gelu_bwd_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(U, n, dA);
}
void launch_vit_add(float* Y, const float* X, int64_t n, cudaStream_t st) {
    vit_add_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(Y, X, n);
}
void launch_vit_gather_tokens(const float* in, int S, int B, int T, int t0, int nt, int D, float* out,
                              cudaStream_t st) {
    const int n4 = B * nt * (D / 4);
    vit_gather_tokens_kernel<<<dim3((n4 + 255) / 256, S), 256, 0, st>>>(in, B, T, t0, nt, D, out);
}

}  // namespace bnn
