// kernels_conv_tc.cu — BF16 tcgen05 implicit-GEMM sampled convolutions for sm_100a
// (SURVEY.md §2.3 K3 fwd, K4 dgrad, K5 wgrad for the ResNet-18-shaped CNN of C3–C5).
//
//   fwd   D[co][pixel]   = Σ_{kh,kw,ci} W_s[co][kh,kw,ci] · X[pixel ⊕ (kh,kw)][ci]
//   dgrad D[ci][in pix]  = Σ_{kh,kw,co} W_s[co][kh,kw,ci] · dY[in pix ⊖ (kh,kw)][co]
//   wgrad D[co][kh,kw,ci]= Σ_pixel dY[pixel][co] · X[pixel ⊕ (kh,kw)][ci]
//
// The A operand (W_s, or dYᵀ for wgrad) is TMA-loaded; the B operand (shifted activation or
// gradient windows, zero-padded at the image border) is gathered by eight producer warps with
// 16-byte cp.async straight into the SWIZZLE_128B UMMA layout and signalled through
// cp.async.mbarrier.arrive. One thread issues tcgen05.mma (M = 128, K = 16 steps) into a
// TMEM accumulator; the epilogue warps read it with tcgen05.ld and fuse bias, residual, ReLU,
// the ReLU mask of the layer input and the bias-gradient partial sums.
#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_conv.cuh"
#include "tc_ptx.cuh"

namespace bnn {

using namespace ptx;

// ============================================================================ W scratch
// Block = one output-channel row co (blockIdx.x) of every sample; thread = column quads of the
// row; μ and σ are loaded once per quad and reused for the S samples.
__global__ void __launch_bounds__(512)
    gen_wscratch_kernel(SampledLayer L, SampleKeys kk, int S, int C, int C_pad, int taps, int K_pad,
                        __nv_bfloat16* __restrict__ out, float* __restrict__ bias_out) {
    const int co = blockIdx.x;
    // blockIdx.y: a group of samples [s_lo, s_hi) (more blocks for layers with few rows)
    const int sg = (S + gridDim.y - 1) / gridDim.y, s_lo = blockIdx.y * sg, s_hi = min(S, s_lo + sg);
    for (int s = s_lo + threadIdx.x; bias_out && s < s_hi; s += blockDim.x) {  // sampled biases b_s, fp32 [S][N]
        bias_out[(int64_t)s * L.N + co] = __fmaf_rn(
            L.sigma[L.off_b + co], eps1(kk.key, kk.step, kk.s0 + s, L.t_b, 0u, (uint32_t)co), L.mu[L.off_b + co]);
    }
    const int kq = K_pad / 4;
    const int Kt = L.K;  // = taps·C
    const int64_t srow = (int64_t)L.N * K_pad;
    __nv_bfloat16* orow = out + (int64_t)co * K_pad;
    for (int qd = threadIdx.x; qd < kq; qd += blockDim.x) {
        const int kp = qd * 4;
        if (C_pad == C) {
            // column kp = tap·C + ci is the parameter column; C % 4 == 0 ⇒ one Philox quad
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f), g = m;
            const bool ok = kp < Kt;
            if (ok) {
                const int64_t i = L.off_w + (int64_t)co * Kt + kp;
                m = __ldg(reinterpret_cast<const float4*>(L.mu + i));
                g = __ldg(reinterpret_cast<const float4*>(L.sigma + i));
            }
#pragma unroll 4
            for (int s = s_lo; s < s_hi; ++s) {  // independent Philox chains: unrolled for ILP
                uint2 v = make_uint2(0u, 0u);
                if (ok) {
                    const float4 e = eps4(kk.key, kk.step, kk.s0 + s, L.t_w, (uint32_t)co, (uint32_t)qd);
                    v = make_uint2(pack_bf16x2(__fmaf_rn(g.x, e.x, m.x), __fmaf_rn(g.y, e.y, m.y)),
                                   pack_bf16x2(__fmaf_rn(g.z, e.z, m.z), __fmaf_rn(g.w, e.w, m.w)));
                }
                *reinterpret_cast<uint2*>(orow + s * srow + kp) = v;
            }
        } else {
            for (int s = s_lo; s < s_hi; ++s) {
                float w[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int tap = (kp + j) / C_pad, ci = (kp + j) % C_pad;
                    if (tap < taps && ci < C) {
                        const int col = tap * C + ci;
                        const int64_t i = L.off_w + (int64_t)co * Kt + col;
                        w[j] = __fmaf_rn(L.sigma[i],
                                         eps1(kk.key, kk.step, kk.s0 + s, L.t_w, (uint32_t)co, (uint32_t)col), L.mu[i]);
                    }
                }
                *reinterpret_cast<uint2*>(orow + s * srow + kp) =
                    make_uint2(pack_bf16x2(w[0], w[1]), pack_bf16x2(w[2], w[3]));
            }
        }
    }
}

void launch_gen_wscratch(const SampledLayer& L, const SampleKeys& kk, int S, int C, int C_pad,
                         int taps, int K_pad, __nv_bfloat16* out, float* bias_out, cudaStream_t st) {
    const int kq = K_pad / 4;
    // balanced blocks: a thread count (multiple of 32, ≤ 512) that divides the row's quads when one
    // exists (a 4608-column row: 384 threads × 3 quads instead of 256 × 4.5), and sample groups that
    // divide S, enough of them for a layer with few rows to fill the GPU (≥ 8 blocks per SM)
    int threads = kq >= 256 ? 256 : ((kq + 31) / 32) * 32;
    for (int t = 512; t >= 128; t -= 32)
        if (kq % t == 0) {
            threads = t;
            break;
        }
    int groups = std::max(1, std::min(S, (8 * kNumSMs + L.N - 1) / L.N));
    while (groups > 1 && S % groups != 0) --groups;
    gen_wscratch_kernel<<<dim3(L.N, groups), std::max(threads, 32), 0, st>>>(L, kk, S, C, C_pad, taps, K_pad, out,
                                                                           bias_out);
}

// ============================================================================ split reduce
// (the SIMT bf16 wgrad of layers whose C is not a multiple of 64: fixed-order sum of splits)
__global__ void wgrad_split_reduce_kernel(const float* __restrict__ part, int nsplit, int64_t n,
                                          int64_t off, float* __restrict__ acc_mu,
                                          float* __restrict__ acc_rho) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float m = 0.0f, r = 0.0f;
        for (int sp = 0; sp < nsplit; ++sp) {  // fixed order ⇒ deterministic
            m += part[(int64_t)sp * 2 * n + i];
            r += part[(int64_t)sp * 2 * n + n + i];
        }
        acc_mu[off + i] += m;
        acc_rho[off + i] += r;
    }
}

// float4 form (n, off multiples of 4): block = 32 column quads × 8 split groups; group g sums the
// splits g, g + 8, … in order (loads of 4 splits in flight), the 8 groups are added in group order
// through shared memory ⇒ deterministic, and 288 blocks for a stage-1 layer instead of 36
__global__ void __launch_bounds__(256) wgrad_split_reduce4_kernel(const float* __restrict__ part, int nsplit, int64_t n,
                                                                  int64_t off, float* __restrict__ acc_mu,
                                                                  float* __restrict__ acc_rho) {
    __shared__ float4 red[2][8][33];
    const int64_t n4 = n / 4;
    const int tx = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + tx;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f), r = m;
    if (i < n4) {
        const float4* pm = reinterpret_cast<const float4*>(part) + i;
        for (int sp0 = g; sp0 < nsplit; sp0 += 32) {
            float4 xm[4], xr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (sp0 + 8 * j < nsplit) {
                    xm[j] = __ldcs(pm + (int64_t)(sp0 + 8 * j) * 2 * n4);
                    xr[j] = __ldcs(pm + (int64_t)(sp0 + 8 * j) * 2 * n4 + n4);
                }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (sp0 + 8 * j < nsplit) {
                    m.x += xm[j].x; m.y += xm[j].y; m.z += xm[j].z; m.w += xm[j].w;
                    r.x += xr[j].x; r.y += xr[j].y; r.z += xr[j].z; r.w += xr[j].w;
                }
        }
    }
    red[0][g][tx] = m;
    red[1][g][tx] = r;
    __syncthreads();
    if (g == 0 && i < n4) {
        for (int k = 1; k < 8; ++k) {
            const float4 a = red[0][k][tx], b = red[1][k][tx];
            m.x += a.x; m.y += a.y; m.z += a.z; m.w += a.w;
            r.x += b.x; r.y += b.y; r.z += b.z; r.w += b.w;
        }
        float4* am = reinterpret_cast<float4*>(acc_mu + off) + i;
        float4* ar = reinterpret_cast<float4*>(acc_rho + off) + i;
        const float4 a0 = *am, b0 = *ar;
        *am = make_float4(a0.x + m.x, a0.y + m.y, a0.z + m.z, a0.w + m.w);
        *ar = make_float4(b0.x + r.x, b0.y + r.y, b0.z + r.z, b0.w + r.w);
    }
}

void launch_wgrad_split_reduce(const float* part, int nsplit, int64_t n, int64_t off, float* acc_mu,
                               float* acc_rho, cudaStream_t st) {
    if (n % 4 == 0 && off % 4 == 0) {
        wgrad_split_reduce4_kernel<<<(int)std::max<int64_t>(1, (n / 4 + 31) / 32), 256, 0, st>>>(part, nsplit, n, off,
                                                                                              acc_mu, acc_rho);
        return;
    }
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8);
    wgrad_split_reduce_kernel<<<std::max(grid, 1), 256, 0, st>>>(part, nsplit, n, off, acc_mu, acc_rho);
}

// ============================================================================ helpers
// bf16 NHWC input with channel padding; aug = 1 applies the PER_SAMPLE crop + flip of
// docs/EPS.md §4 (keyed by global sample and global example), aug = 0 copies x (S = 1).
__global__ void input_bf16_kernel(const float* __restrict__ x, int B, int H, int W, int C,
                                  int C_pad, int aug, EpsKey key, uint32_t step, uint32_t s0,
                                  int b_off, __nv_bfloat16* __restrict__ out) {
    const int b = blockIdx.x, s = blockIdx.y;
    int dx = 4, dy = 4, flip = 0;
    if (aug) {
        const uint4 y = philox10(make_uint4(0u, (uint32_t)(b_off + b), (4095u << 20) | (s0 + s), step), key);
        dx = (int)(y.x % 9u);
        dy = (int)(y.y % 9u);
        flip = (int)(y.z & 1u);
    }
    const float* src = x + (int64_t)b * H * W * C;
    __nv_bfloat16* dst = out + ((int64_t)s * B + b) * H * W * C_pad;
    if (C_pad == 8 && C <= 8) {  // thread = pixel: its 8 (padded) channels as one 16-byte store
        for (int pix = threadIdx.x; pix < H * W; pix += blockDim.x) {
            const int r = pix / W, cc = pix - r * W;
            const int jj = flip ? W - 1 - cc : cc;
            const int si = r + dy - 4, sj = jj + dx - 4;
            const bool in = si >= 0 && si < H && sj >= 0 && sj < W;
            float v[8];
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) v[ch] = (in && ch < C) ? src[((int64_t)si * W + sj) * C + ch] : 0.0f;
            *reinterpret_cast<uint4*>(dst + (int64_t)pix * 8) =
                make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
        }
        return;
    }
    for (int i = threadIdx.x; i < H * W * C_pad; i += blockDim.x) {
        const int ch = i % C_pad, pix = i / C_pad, r = pix / W, cc = pix % W;
        const int jj = flip ? W - 1 - cc : cc;
        const int si = r + dy - 4, sj = jj + dx - 4;
        const float v = (ch < C && si >= 0 && si < H && sj >= 0 && sj < W)
                            ? src[((int64_t)si * W + sj) * C + ch]
                            : 0.0f;
        dst[i] = __float2bfloat16_rn(v);
    }
}

void launch_input_bf16(const float* x, int S, int B, int H, int W, int C, int C_pad, int aug,
                       uint64_t seed, uint32_t step, uint32_t s0, int b_off, __nv_bfloat16* out,
                       cudaStream_t st) {
    input_bf16_kernel<<<dim3(B, S), 256, 0, st>>>(x, B, H, W, C, C_pad, aug, make_key(seed), step, s0,
                                                  b_off, out);
}

__global__ void gap_fwd_bf16_kernel(const __nv_bfloat16* __restrict__ y, int R, int HW, int C,
                                    __nv_bfloat16* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R * C) return;
    const int r = i / C, ch = i % C;
    float acc = 0.0f;
    for (int p = 0; p < HW; ++p) acc += __bfloat162float(y[((int64_t)r * HW + p) * C + ch]);
    out[i] = __float2bfloat16_rn(acc / HW);
}

void launch_gap_fwd_bf16(const __nv_bfloat16* y, int R, int HW, int C, __nv_bfloat16* out,
                         cudaStream_t st) {
    gap_fwd_bf16_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(y, R, HW, C, out);
}

__global__ void gap_bwd_bf16_kernel(const __nv_bfloat16* __restrict__ gpool, int ldg,
                                    const __nv_bfloat16* __restrict__ y, int R, int HW, int C,
                                    __nv_bfloat16* __restrict__ gy, float* __restrict__ part) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R * C) return;
    const int r = i / C, ch = i % C;
    const float g = __bfloat162float(gpool[(int64_t)r * ldg + ch]) / HW;
    float acc = 0.0f;
    for (int p = 0; p < HW; ++p) {
        const int64_t o = ((int64_t)r * HW + p) * C + ch;
        const float v = __bfloat162float(y[o]) > 0.0f ? g : 0.0f;
        gy[o] = __float2bfloat16_rn(v);
        acc += v;
    }
    part[i] = acc;
}

void launch_gap_bwd_bf16(const __nv_bfloat16* gpool, int ldg, const __nv_bfloat16* y, int R, int HW,
                         int C, __nv_bfloat16* gy, float* part, cudaStream_t st) {
    gap_bwd_bf16_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(gpool, ldg, y, R, HW, C, gy, part);
}

// SIMT wgrad on bf16 operands (the stem: C_in = 3, K = 27) — 64 co × 64 cols per CTA
__global__ void __launch_bounds__(256) conv_wgrad_simt_bf16_kernel(
    SampledLayer L, SampleKeys kk, int S, ConvShape c, int C_pad, const __nv_bfloat16* __restrict__ G,
    int64_t sG, const __nv_bfloat16* __restrict__ X, int64_t sX, float scale,
    float* __restrict__ part, int nsplit) {
    __shared__ float Gs[16][68];
    __shared__ float Xs[16][68];
    const int col0 = blockIdx.x * 64, co0 = blockIdx.y * 64;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int npix = c.B * c.OH * c.OW, Kt = c.k * c.k * c.C;
    const int gcol = col0 + (tid & 63);
    const int gci = gcol % c.C, gkhw = gcol / c.C, gkh = gkhw / c.k, gkw = gkhw % c.k;
    float am[4][4] = {}, ar[4][4] = {};
    const int per = (npix + nsplit - 1) / nsplit;
    const int pbeg = blockIdx.z * per, pend = min(npix, pbeg + per);
    for (int s = 0; s < S; ++s) {
        const __nv_bfloat16* Gg = G + s * sG;
        const __nv_bfloat16* Xg = X + s * sX;
        float d[4][4] = {};
        for (int p0 = pbeg; p0 < pend; p0 += 16) {
            const int pr = tid >> 6;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int p = p0 + 4 * pr + j;
                const int co = co0 + (tid & 63);
                Gs[4 * pr + j][tid & 63] =
                    (p < pend && co < c.CO) ? __bfloat162float(Gg[(int64_t)p * c.CO + co]) : 0.0f;
                float v = 0.0f;
                if (p < pend && gcol < Kt) {
                    const int n = p / (c.OH * c.OW), rem = p % (c.OH * c.OW);
                    const int ih = (rem / c.OW) * c.stride + gkh - c.pad;
                    const int iw = (rem % c.OW) * c.stride + gkw - c.pad;
                    if (ih >= 0 && ih < c.H && iw >= 0 && iw < c.W)
                        v = __bfloat162float(Xg[(((int64_t)n * c.H + ih) * c.W + iw) * C_pad + gci]);
                }
                Xs[4 * pr + j][tid & 63] = v;
            }
            __syncthreads();
#pragma unroll
            for (int qq = 0; qq < 16; ++qq) {
                float g[4], x[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) g[i] = Gs[qq][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = Xs[qq][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) d[i][j] = fmaf(g[i], x[j], d[i][j]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int co = co0 + ty * 4 + i;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int col = col0 + tx * 4 + j;
                if (co >= c.CO || col >= Kt) continue;
                am[i][j] += d[i][j];
                ar[i][j] = fmaf(d[i][j], eps1(kk.key, kk.step, kk.s0 + s, L.t_w, co, col), ar[i][j]);
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
            const int64_t n = (int64_t)c.CO * Kt;
            const int64_t o = (int64_t)blockIdx.z * 2 * n + (int64_t)co * Kt + col;
            part[o] = scale * am[i][j];
            part[o + n] = scale * ar[i][j];
        }
    }
}

void launch_conv_wgrad_simt_bf16(const SampledLayer& L, const SampleKeys& kk, int S,
                                 const ConvShape& c, int C_pad, const __nv_bfloat16* G, int64_t sG,
                                 const __nv_bfloat16* X, int64_t sX, float scale, float* part,
                                 int nsplit, cudaStream_t st) {
    const int Kt = c.k * c.k * c.C;
    dim3 grid((Kt + 63) / 64, (c.CO + 63) / 64, nsplit);
    conv_wgrad_simt_bf16_kernel<<<grid, 256, 0, st>>>(L, kk, S, c, C_pad, G, sG, X, sX, scale, part,
                                                      nsplit);
}

}  // namespace bnn
