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
__global__ void vit_embed_kernel(const float* __restrict__ E, const float* __restrict__ cls,
                                 const float* __restrict__ pos, int B, int T, int D, float* __restrict__ X) {
    const int64_t n = (int64_t)B * T * D;
    const int s = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(i % D), t = (int)((i / D) % T), b = (int)(i / ((int64_t)T * D));
        const float v = t == 0 ? cls[(int64_t)s * D + d] : E[(((int64_t)s * B + b) * (T - 1) + t - 1) * D + d];
        X[(int64_t)s * n + i] = v + pos[(int64_t)s * T * D + (int64_t)t * D + d];
    }
}

void launch_vit_embed(const float* E, const float* cls, const float* pos, int S, int B, int T, int D, float* X,
                      cudaStream_t st) {
    vit_embed_kernel<<<dim3(256, S), 256, 0, st>>>(E, cls, pos, B, T, D, X);
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
void launch_vit_ln_fwd(const float* X, int S, int rows, int64_t ld, int64_t sX, int D, const float* g, const float* b,
                       __nv_bfloat16* Y, int64_t ldy, int64_t sY, float* stats, cudaStream_t st) {
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
void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, float* O, float* A,
                         cudaStream_t st) {
    attn_fwd_t(QKV, S, B, T, D, heads, O, A, st);
}
void launch_vit_attn_fwd(const float* QKV, int S, int B, int T, int D, int heads, __nv_bfloat16* O, float* A,
                         cudaStream_t st) {
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
void launch_vit_attn_bwd(const float* QKV, const float* A, const __nv_bfloat16* dO, int S, int B, int T, int D,
                         int heads, float* dQKV, cudaStream_t st) {
    attn_bwd_t(QKV, A, dO, S, B, T, D, heads, dQKV, st);
}

// ------------------------------------------------------------------------ elementwise
__device__ __forceinline__ float gelu_f(float u) { return 0.5f * u * (1.0f + erff(u * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_df(float u) {
    return 0.5f * (1.0f + erff(u * 0.70710678118654752f)) + u * 0.39894228040143268f * __expf(-0.5f * u * u);
}

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
    const int64_t n = (int64_t)B * nt * D;
    const int s = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(i % D), k = (int)((i / D) % nt), b = (int)(i / ((int64_t)nt * D));
        out[(int64_t)s * n + i] = in[(((int64_t)s * B + b) * T + t0 + k) * D + d];
    }
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
    vit_gather_tokens_kernel<<<dim3(256, S), 256, 0, st>>>(in, B, T, t0, nt, D, out);
}

}  // namespace bnn
