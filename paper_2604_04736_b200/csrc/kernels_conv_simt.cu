// kernels_conv_simt.cu — FP32 SIMT sampled convolutions (K11 for the ResNet-18-shaped CNN,
// FP32 parity mode) and the image-path elementwise kernels (K9 augmentation, GAP, masks).
//
// Convolution (NHWC activations, OHWI weights viewed as [c_out, kh·kw·c_in]):
//   fwd   Y[n,oh,ow,co] = act(Σ_{kh,kw,ci} W_s[co,kh,kw,ci]·X[n, oh·st+kh−p, ow·st+kw−p, ci]
//                             + b_s[co] (+ R[n,oh,ow,co]))
//   dgrad dX[n,ih,iw,ci] (+)= Σ_{co,kh,kw} G[n,oh,ow,co]·W_s[co,kh,kw,ci],  oh·st = ih+p−kh
//   wgrad acc_μ += scale·Σ_s dW_s,  acc_ρ += scale·Σ_s dW_s ⊙ ε_s,
//         dW_s[co,kh,kw,ci] = Σ_{n,oh,ow} G[n,oh,ow,co]·X[n, oh·st+kh−p, ow·st+kw−p, ci]
// W_s = fma(σ, ε_s, μ) is generated per tile from EPS-v1 exactly as in the MLP kernels.
#include <algorithm>

#include "common.cuh"
#include "kernels_conv.cuh"

namespace bnn {

namespace {
constexpr int TT = 64, TKc = 16;

__device__ __forceinline__ float gen_w(const SampledLayer& L, const float4& e, int j, int64_t i) {
    return __fmaf_rn(L.sigma[i], eps_get(e, j), L.mu[i]);
}
}  // namespace

// ---------------------------------------------------------------- fwd
__global__ void __launch_bounds__(256) conv_fwd_fp32_kernel(SampledLayer L, SampleKeys kk,
                                                            ConvShape c,
                                                            const float* __restrict__ X,
                                                            int64_t sX,
                                                            const float* __restrict__ R,
                                                            int64_t sR, float* __restrict__ Y,
                                                            int64_t sY, int relu) {
    __shared__ float Ws[TKc][TT + 4];  // [k][co]
    __shared__ float Xs[TKc][TT + 4];  // [k][pixel]
    __shared__ float bias[TT];
    const int co0 = blockIdx.x * TT, p0 = blockIdx.y * TT, s = blockIdx.z;
    const uint32_t sg = kk.s0 + s;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int npix = c.B * c.OH * c.OW, Kt = c.k * c.k * c.C;
    const float* Xg = X + s * sX;
    float acc[4][4] = {};
    // gather geometry of this thread's pixel (fixed across the K loop)
    const int gp = p0 + (tid & 63);
    const int gn = gp / (c.OH * c.OW), grem = gp % (c.OH * c.OW);
    const int goh = grem / c.OW, gow = grem % c.OW;
    for (int k0 = 0; k0 < Kt; k0 += TKc) {
        {
            const int r = tid >> 2, kq = tid & 3, co = co0 + r, kb = k0 + 4 * kq;
            float w[4] = {0.f, 0.f, 0.f, 0.f};
            if (co < c.CO && kb < Kt) {
                const float4 e = eps4(kk.key, kk.step, sg, L.t_w, co, kb >> 2);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (kb + j < Kt) w[j] = gen_w(L, e, j, L.off_w + (int64_t)co * Kt + kb + j);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) Ws[4 * kq + j][r] = w[j];
        }
        {
            const int kr = tid >> 6;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int kidx = k0 + 4 * kr + j;
                float v = 0.0f;
                if (gp < npix && kidx < Kt) {
                    const int ci = kidx % c.C, khw = kidx / c.C, kh = khw / c.k, kw = khw % c.k;
                    const int ih = goh * c.stride + kh - c.pad, iw = gow * c.stride + kw - c.pad;
                    if (ih >= 0 && ih < c.H && iw >= 0 && iw < c.W)
                        v = Xg[(((int64_t)gn * c.H + ih) * c.W + iw) * c.C + ci];
                }
                Xs[4 * kr + j][tid & 63] = v;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TKc; ++q) {
            float w[4], x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = Ws[q][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = Xs[q][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(w[i], x[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (tid < TT) {
        const int co = co0 + tid;
        bias[tid] = co < c.CO ? __fmaf_rn(L.sigma[L.off_b + co], eps1(kk.key, kk.step, sg, L.t_b, 0, co),
                                          L.mu[L.off_b + co])
                              : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = co0 + ty * 4 + i;
        if (co >= c.CO) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int p = p0 + tx * 4 + j;
            if (p >= npix) continue;
            const int64_t o = (int64_t)p * c.CO + co;
            float v = acc[i][j] + bias[ty * 4 + i];
            if (R) v += R[s * sR + o];
            if (relu) v = fmaxf(v, 0.0f);
            Y[s * sY + o] = v;
        }
    }
}

void launch_conv_fwd_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                          const float* X, int64_t sX, const float* R, int64_t sR, float* Y,
                          int64_t sY, bool relu, cudaStream_t st) {
    const int npix = c.B * c.OH * c.OW;
    dim3 grid((c.CO + TT - 1) / TT, (npix + TT - 1) / TT, S);
    conv_fwd_fp32_kernel<<<grid, 256, 0, st>>>(L, kk, c, X, sX, R, sR, Y, sY, relu ? 1 : 0);
}

// ---------------------------------------------------------------- dgrad
__global__ void __launch_bounds__(256) conv_dgrad_fp32_kernel(SampledLayer L, SampleKeys kk,
                                                              ConvShape c,
                                                              const float* __restrict__ G,
                                                              int64_t sG, float* __restrict__ dX,
                                                              int64_t sdX, int accumulate) {
    __shared__ float Ws[TKc][TT + 4];  // [co][ci]
    __shared__ float Gs[TKc][TT + 4];  // [co][input pixel]
    const int ci0 = blockIdx.x * TT, p0 = blockIdx.y * TT, s = blockIdx.z;
    const uint32_t sg = kk.s0 + s;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int npix = c.B * c.H * c.W, Kt = c.k * c.k * c.C;
    const float* Gg = G + s * sG;
    const int gp = p0 + (tid & 63);
    const int gn = gp / (c.H * c.W), grem = gp % (c.H * c.W);
    const int gih = grem / c.W, giw = grem % c.W;
    float acc[4][4] = {};
    for (int kh = 0; kh < c.k; ++kh)
        for (int kw = 0; kw < c.k; ++kw) {
            // output position feeding this input pixel through tap (kh, kw)
            const int th = gih + c.pad - kh, tw = giw + c.pad - kw;
            const bool ok = gp < npix && th >= 0 && tw >= 0 && th % c.stride == 0 &&
                            tw % c.stride == 0 && th / c.stride < c.OH && tw / c.stride < c.OW;
            const int64_t gbase =
                ok ? (((int64_t)gn * c.OH + th / c.stride) * c.OW + tw / c.stride) * c.CO : 0;
            for (int c0 = 0; c0 < c.CO; c0 += TKc) {
                {
                    const int r = tid >> 4, cq = tid & 15, co = c0 + r, ci = ci0 + 4 * cq;
                    float w[4] = {0.f, 0.f, 0.f, 0.f};
                    if (co < c.CO && ci < c.C) {
                        const int col = (kh * c.k + kw) * c.C + ci;
                        const float4 e = eps4(kk.key, kk.step, sg, L.t_w, co, col >> 2);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (ci + j < c.C) w[j] = gen_w(L, e, j, L.off_w + (int64_t)co * Kt + col + j);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) Ws[r][4 * cq + j] = w[j];
                }
                {
                    const int cr = tid >> 6;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int co = c0 + 4 * cr + j;
                        Gs[4 * cr + j][tid & 63] = (ok && co < c.CO) ? Gg[gbase + co] : 0.0f;
                    }
                }
                __syncthreads();
#pragma unroll
                for (int q = 0; q < TKc; ++q) {
                    float w[4], g[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) w[i] = Ws[q][ty * 4 + i];
#pragma unroll
                    for (int j = 0; j < 4; ++j) g[j] = Gs[q][tx * 4 + j];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(w[i], g[j], acc[i][j]);
                }
                __syncthreads();
            }
        }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = ci0 + ty * 4 + i;
        if (ci >= c.C) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int p = p0 + tx * 4 + j;
            if (p >= npix) continue;
            float* o = dX + s * sdX + (int64_t)p * c.C + ci;
            *o = accumulate ? *o + acc[i][j] : acc[i][j];
        }
    }
}

void launch_conv_dgrad_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                            const float* G, int64_t sG, float* dX, int64_t sdX, bool accumulate,
                            cudaStream_t st) {
    const int npix = c.B * c.H * c.W;
    dim3 grid((c.C + TT - 1) / TT, (npix + TT - 1) / TT, S);
    conv_dgrad_fp32_kernel<<<grid, 256, 0, st>>>(L, kk, c, G, sG, dX, sdX, accumulate ? 1 : 0);
}

// ---------------------------------------------------------------- wgrad + sample accumulation
__global__ void __launch_bounds__(256) conv_wgrad_fp32_kernel(
    SampledLayer L, SampleKeys kk, int S, ConvShape c, const float* __restrict__ G, int64_t sG,
    const float* __restrict__ X, int64_t sX, float scale, float* __restrict__ acc_mu,
    float* __restrict__ acc_rho) {
    __shared__ float Gs[TKc][TT + 4];  // [pixel][co]
    __shared__ float Xs[TKc][TT + 4];  // [pixel][col]
    const int col0 = blockIdx.x * TT, co0 = blockIdx.y * TT;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int npix = c.B * c.OH * c.OW, Kt = c.k * c.k * c.C;
    // this thread's gather column (fixed)
    const int gcol = col0 + (tid & 63);
    const int gci = gcol % c.C, gkhw = gcol / c.C, gkh = gkhw / c.k, gkw = gkhw % c.k;
    float am[4][4] = {}, ar[4][4] = {};
    for (int s = 0; s < S; ++s) {
        const float* Gg = G + s * sG;
        const float* Xg = X + s * sX;
        float d[4][4] = {};
        for (int p0 = 0; p0 < npix; p0 += TKc) {
            {
                const int pr = tid >> 6;  // 0..3
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int p = p0 + 4 * pr + j;
                    const int co = co0 + (tid & 63);
                    Gs[4 * pr + j][tid & 63] = (p < npix && co < c.CO) ? Gg[(int64_t)p * c.CO + co] : 0.0f;
                    float v = 0.0f;
                    if (p < npix && gcol < Kt) {
                        const int n = p / (c.OH * c.OW), rem = p % (c.OH * c.OW);
                        const int ih = (rem / c.OW) * c.stride + gkh - c.pad;
                        const int iw = (rem % c.OW) * c.stride + gkw - c.pad;
                        if (ih >= 0 && ih < c.H && iw >= 0 && iw < c.W)
                            v = Xg[(((int64_t)n * c.H + ih) * c.W + iw) * c.C + gci];
                    }
                    Xs[4 * pr + j][tid & 63] = v;
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < TKc; ++q) {
                float g[4], x[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) g[i] = Gs[q][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = Xs[q][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) d[i][j] = fmaf(g[i], x[j], d[i][j]);
            }
            __syncthreads();
        }
        const int kb = col0 + tx * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int co = co0 + ty * 4 + i;
            if (co >= c.CO || kb >= Kt) continue;
            const float4 e = eps4(kk.key, kk.step, kk.s0 + s, L.t_w, co, kb >> 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                am[i][j] += d[i][j];
                ar[i][j] = fmaf(d[i][j], eps_get(e, j), ar[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = co0 + ty * 4 + i;
        if (co >= c.CO) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = col0 + tx * 4 + j;
            if (col >= Kt) continue;
            const int64_t o = L.off_w + (int64_t)co * Kt + col;
            acc_mu[o] += scale * am[i][j];
            acc_rho[o] += scale * ar[i][j];
        }
    }
}

void launch_conv_wgrad_fp32(const SampledLayer& L, const SampleKeys& kk, int S, const ConvShape& c,
                            const float* G, int64_t sG, const float* X, int64_t sX, float scale,
                            float* acc_mu, float* acc_rho, cudaStream_t st) {
    const int Kt = c.k * c.k * c.C;
    dim3 grid((Kt + TT - 1) / TT, (c.CO + TT - 1) / TT);
    conv_wgrad_fp32_kernel<<<grid, 256, 0, st>>>(L, kk, S, c, G, sG, X, sX, scale, acc_mu, acc_rho);
}

// ---------------------------------------------------------------- elementwise helpers
__global__ void mask_kernel(float* __restrict__ g, const float* __restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!(y[i] > 0.0f)) g[i] = 0.0f;
}
void launch_relu_mask(float* g, const float* y, int64_t n, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
    mask_kernel<<<std::max(grid, 1), 256, 0, st>>>(g, y, n);
}

__global__ void add_kernel(float* __restrict__ d, const float* __restrict__ a, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] += a[i];
}
void launch_add(float* dst, const float* src, int64_t n, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
    add_kernel<<<std::max(grid, 1), 256, 0, st>>>(dst, src, n);
}

// global average pool: out[r][c] = mean_hw y[r][hw][c], r over S·B images
__global__ void gap_fwd_kernel(const float* __restrict__ y, int R, int HW, int C,
                               float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R * C) return;
    const int r = i / C, ch = i % C;
    float acc = 0.0f;
    for (int p = 0; p < HW; ++p) acc += y[((int64_t)r * HW + p) * C + ch];
    out[i] = acc / HW;
}
void launch_gap_fwd(const float* y, int R, int HW, int C, float* out, cudaStream_t st) {
    gap_fwd_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(y, R, HW, C, out);
}
__global__ void gap_bwd_kernel(const float* __restrict__ gp, int R, int HW, int C,
                               float* __restrict__ gy) {
    const int64_t n = (int64_t)R * HW * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ch = (int)(i % C);
        const int64_t r = i / ((int64_t)HW * C);
        gy[i] = gp[r * C + ch] / HW;
    }
}
void launch_gap_bwd(const float* gpool, int R, int HW, int C, float* gy, cudaStream_t st) {
    const int64_t n = (int64_t)R * HW * C;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
    gap_bwd_kernel<<<std::max(grid, 1), 256, 0, st>>>(gpool, R, HW, C, gy);
}

// K9: per-(global sample, global example) random crop (zero pad 4) + horizontal flip,
// keyed by EPS-v1 tag t = 4095 (docs/EPS.md §4, R11). out[s][b] ← x[b].
__global__ void augment_kernel(const float* __restrict__ x, int B, int H, int W, int C,
                               EpsKey key, uint32_t step, uint32_t s0, int b_off,
                               float* __restrict__ out) {
    const int b = blockIdx.x, s = blockIdx.y;
    __shared__ int prm[3];
    if (threadIdx.x == 0) {
        const uint4 y = philox10(make_uint4(0u, (uint32_t)(b_off + b), (4095u << 20) | (s0 + s), step), key);
        prm[0] = (int)(y.x % 9u);
        prm[1] = (int)(y.y % 9u);
        prm[2] = (int)(y.z & 1u);
    }
    __syncthreads();
    const int dx = prm[0], dy = prm[1], flip = prm[2];
    const float* src = x + (int64_t)b * H * W * C;
    float* dst = out + ((int64_t)s * B + b) * H * W * C;
    for (int i = threadIdx.x; i < H * W * C; i += blockDim.x) {
        const int ch = i % C, pix = i / C, r = pix / W, cc = pix % W;
        const int jj = flip ? W - 1 - cc : cc;
        const int si = r + dy - 4, sj = jj + dx - 4;
        dst[i] = (si >= 0 && si < H && sj >= 0 && sj < W) ? src[((int64_t)si * W + sj) * C + ch] : 0.0f;
    }
}
void launch_augment(const float* x, int S, int B, int H, int W, int C, uint64_t seed,
                    uint32_t step, uint32_t s0, int b_off, float* out, cudaStream_t st) {
    augment_kernel<<<dim3(B, S), 256, 0, st>>>(x, B, H, W, C, make_key(seed), step, s0, b_off, out);
}

}  // namespace bnn
