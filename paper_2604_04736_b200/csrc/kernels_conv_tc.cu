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
__global__ void __launch_bounds__(256)
    gen_wscratch_kernel(SampledLayer L, SampleKeys kk, int S, int C, int C_pad, int taps, int K_pad,
                        __nv_bfloat16* __restrict__ out, float* __restrict__ bias_out) {
    const int co = blockIdx.x;
    for (int s = threadIdx.x; bias_out && s < S; s += blockDim.x) {  // sampled biases b_s, fp32 [S][N]
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
            for (int s = 0; s < S; ++s) {  // independent Philox chains: unrolled for ILP
                uint2 v = make_uint2(0u, 0u);
                if (ok) {
                    const float4 e = eps4(kk.key, kk.step, kk.s0 + s, L.t_w, (uint32_t)co, (uint32_t)qd);
                    v = make_uint2(pack_bf16x2(__fmaf_rn(g.x, e.x, m.x), __fmaf_rn(g.y, e.y, m.y)),
                                   pack_bf16x2(__fmaf_rn(g.z, e.z, m.z), __fmaf_rn(g.w, e.w, m.w)));
                }
                *reinterpret_cast<uint2*>(orow + s * srow + kp) = v;
            }
        } else {
            for (int s = 0; s < S; ++s) {
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
    const int threads = kq >= 256 ? 256 : ((kq + 31) / 32) * 32;
    gen_wscratch_kernel<<<L.N, std::max(threads, 32), 0, st>>>(L, kk, S, C, C_pad, taps, K_pad, out, bias_out);
}

// ============================================================================ fwd / dgrad
namespace cv {
constexpr int kProdWarps = 8;                    // gather producers + epilogue
constexpr int kThreads = (kProdWarps + 2) * 32;  // + MMA warp + TMA warp
constexpr int kStages = 2;
constexpr int kAStage = 128 * 64 * 2;  // 16 KB
constexpr int kBStage = 256 * 64 * 2;  // 32 KB
constexpr int kSmem = 1024 + kStages * (kAStage + kBStage) + 256 + 128 * 4 + 64;
}  // namespace cv

template <int MODE>  // 0 fwd, 1 dgrad
__global__ void __launch_bounds__(cv::kThreads, 2)
    conv_tc_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap bmap,
                   const ConvTcArgs a) {
    using namespace cv;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
    float* sbias = reinterpret_cast<float*>(bars + 32);
    int* staps = reinterpret_cast<int*>(sbias + 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int m0 = blockIdx.x * 128;
    int s, cls = 0, ncls = 1;
    if (MODE == 1) {
        ncls = a.stride * a.stride;
        s = blockIdx.z / ncls;
        cls = blockIdx.z % ncls;
    } else {
        s = blockIdx.z;
    }
    const int ph = cls / a.stride, pw = cls % a.stride;
    // pixel space of this launch: fwd → output pixels; dgrad → input pixels of class (ph, pw)
    const int PH = MODE == 0 ? a.OH : a.H / a.stride, PW = MODE == 0 ? a.OW : a.W / a.stride;
    const int npix = a.B * PH * PW;
    const int p0 = blockIdx.y * 256;
    const uint32_t sg = a.kk.s0 + s;
    const SampledLayer& L = a.L;
    const int M = MODE == 0 ? a.CO : a.C;

    // K blocks: fwd → K_pad/64; dgrad → (valid taps of the class) × CO/64
    int ntaps = 0;
    if (MODE == 1) {
        for (int kh = 0; kh < a.k; ++kh)
            for (int kw = 0; kw < a.k; ++kw)
                if ((ph + a.pad - kh) % a.stride == 0 && (pw + a.pad - kw) % a.stride == 0) {
                    // ((ph + pad − kh) may be negative: C++ % keeps the sign, 0 test is exact)
                    if (tid == 0) staps[ntaps] = kh * a.k + kw;
                    ++ntaps;
                }
    }
    const int cblocks = (a.CO + 63) / 64;
    const int nkb = MODE == 0 ? a.K_pad / 64 : ntaps * cblocks;

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], a.tma_b ? 1 : kProdWarps * 32 + 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_fence_init();
    }
    if (warp == kProdWarps) tmem_alloc(tslot, 256);
    if (MODE == 0 && tid < 128) {
        const int co = m0 + tid;
        sbias[tid] = co < L.N ? __fmaf_rn(L.sigma[L.off_b + co],
                                          eps1(a.kk.key, a.kk.step, sg, L.t_b, 0u, (uint32_t)co),
                                          L.mu[L.off_b + co])
                              : 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == kProdWarps) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0 && nkb > 0) {
            const uint32_t idesc = idesc_bf16(128, 256, MODE == 1 ? 1 : 0, 0);
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % kStages;
                const uint32_t ph2 = (kb / kStages) & 1;
                mbar_wait_sleep(&full[st], ph2);
                fence_proxy_async_smem();  // cp.async (generic proxy) writes → tensor-core reads
                tc_fence_after();
                const uint32_t aBase = smem_u32(sA + st * kAStage);
                const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint64_t ad = MODE == 0 ? sdesc_sw128(aBase + 32 * q, 16, 1024)
                                                  : sdesc_sw128(aBase + 2048 * q, 8192, 1024);
                    const uint64_t bd = sdesc_sw128(bBase + 32 * q, 16, 1024);
                    mma_bf16(tmem, ad, bd, idesc, (kb | q) != 0 ? 1u : 0u);
                }
                mma_commit(&empty[st]);
            }
            mma_commit(tfull);
        }
        __syncwarp();
    } else if (warp == kProdWarps + 1) {
        // ------------------------------------------------ TMA producer: A (and B for stride 1)
        if (lane == 0 && nkb > 0) {
            tma_prefetch_desc(&wmap);
            if (a.tma_b) tma_prefetch_desc(&bmap);
            // tile origin in (image, row) of the pixel space (stride-1 tiles are row-aligned boxes)
            const int n0 = p0 / (PH * PW), y0 = (p0 - n0 * (PH * PW)) / PW;
            const int sb = a.src_stride_s == 0 ? 0 : s;
            const int cpb_t = a.C_pad >> 6;
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % kStages;
                const uint32_t ph2 = (kb / kStages) & 1;
                mbar_wait_sleep(&empty[st], ph2 ^ 1);
                mbar_arrive_expect_tx(&full[st], kAStage + (a.tma_b ? kBStage : 0));
                uint8_t* dst = sA + st * kAStage;
                if (MODE == 0) {
                    tma_load_3d(&wmap, &full[st], dst, kb * 64, m0, s);
                    if (a.tma_b) {
                        const int tap = kb / cpb_t, c0 = (kb - tap * cpb_t) * 64;
                        const int kh = tap / a.k, kw = tap - kh * a.k;
                        tma_load_5d(&bmap, &full[st], sB + st * kBStage, c0, kw - a.pad, y0 + kh - a.pad,
                                    n0, sb);
                    }
                } else {
                    const int ti = kb / cblocks, tap = staps[ti], cb = kb - ti * cblocks;
                    tma_load_4d(&wmap, &full[st], dst, m0, tap, cb * 64, s);
                    tma_load_4d(&wmap, &full[st], dst + 8192, m0 + 64, tap, cb * 64, s);
                    if (a.tma_b) {
                        const int kh = tap / a.k, kw = tap - kh * a.k;
                        tma_load_5d(&bmap, &full[st], sB + st * kBStage, cb * 64, a.pad - kw,
                                    y0 + a.pad - kh, n0, s);
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ gather producers: row = pixel tid
        const int pix = p0 + tid;
        const bool pvalid = pix < npix;
        const int pn = pvalid ? pix / (PH * PW) : 0;
        const int prem = pvalid ? pix % (PH * PW) : 0;
        const int py = MODE == 0 ? prem / PW : (prem / PW) * a.stride + ph;
        const int px = MODE == 0 ? prem % PW : (prem % PW) * a.stride + pw;
        const __nv_bfloat16* srcs = a.src + s * a.src_stride_s;
        const uint32_t rowoff = tid * 128;
        const uint32_t sw = tid & 7;
        const int cpb = a.C_pad >> 6;  // 64-channel blocks per tap (0 for the 8-channel stem input)
        for (int kb = 0; kb < (a.tma_b ? 0 : nkb); ++kb) {
            const int st = kb % kStages;
            const uint32_t ph2 = (kb / kStages) & 1;
            mbar_wait(&empty[st], ph2 ^ 1);
            const uint32_t base = smem_u32(sB + st * kBStage) + rowoff;
            if (MODE == 0 && cpb == 0) {
                // stem: 8 taps × 8 channels per K block
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int tap = kb * 8 + j;
                    const int kh = tap / a.k, kw = tap - (tap / a.k) * a.k;
                    const int iy = py * a.stride + kh - a.pad, ix = px * a.stride + kw - a.pad;
                    const bool ok = pvalid && tap < a.k * a.k && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                    const __nv_bfloat16* g =
                        ok ? srcs + (((int64_t)pn * a.H + iy) * a.W + ix) * a.C_pad : srcs;
                    cp_async16(base + ((j ^ sw) << 4), g, ok ? 16u : 0u);
                }
            } else {
                // one tap and 64 consecutive channels per K block: one address, 8 chunks
                int kh, kw, c0;
                if (MODE == 0) {
                    const int tap = kb / cpb;
                    c0 = (kb - tap * cpb) * 64;
                    kh = tap / a.k;
                    kw = tap - kh * a.k;
                } else {
                    const int ti = kb / cblocks;
                    const int tap = staps[ti];
                    c0 = (kb - ti * cblocks) * 64;
                    kh = tap / a.k;
                    kw = tap - kh * a.k;
                }
                bool ok;
                const __nv_bfloat16* g = srcs;
                if (MODE == 0) {
                    const int iy = py * a.stride + kh - a.pad, ix = px * a.stride + kw - a.pad;
                    ok = pvalid && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                    if (ok) g = srcs + (((int64_t)pn * a.H + iy) * a.W + ix) * a.C_pad + c0;
                } else {
                    const int ty = py + a.pad - kh, tx = px + a.pad - kw;
                    const int oy = ty / a.stride, ox = tx / a.stride;
                    ok = pvalid && ty >= 0 && tx >= 0 && oy < a.OH && ox < a.OW;
                    if (ok) g = srcs + (((int64_t)pn * a.OH + oy) * a.OW + ox) * a.CO + c0;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) cp_async16(base + ((j ^ sw) << 4), g + 8 * j, ok ? 16u : 0u);
            }
            cp_async_mbar_arrive(&full[st]);
        }
        // ------------------------------------------------ epilogue
        const int q = warp & 3, h = warp >> 2;
        const int row = 32 * q + lane, m = m0 + row;
        const bool mvalid = m < M;
        const float bias = MODE == 0 ? sbias[row] : 0.0f;
        float part = 0.0f;
        if (nkb > 0) {
            mbar_wait_sleep(tfull, 0);
            tc_fence_after();
        }
        __nv_bfloat16* outs = a.out + s * a.out_stride_s;
        for (int c = h; c < 16; c += 2) {
            float v[16];
            __syncwarp();
            if (nkb > 0) {
                tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + c * 16, v);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.0f;
            }
            if (!mvalid) continue;
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const int pp = p0 + c * 16 + j;
                if (pp >= npix) break;
                if (MODE == 0) {
                    const int64_t o = (int64_t)pp * a.CO + m;
                    float z = v[j] + bias;
                    if (a.res) z += __bfloat162float(a.res[s * a.res_stride_s + o]);
                    if (a.relu) z = fmaxf(z, 0.0f);
                    outs[o] = __float2bfloat16_rn(z);
                } else {
                    int64_t o;
                    if (a.stride == 1) {
                        o = (int64_t)pp * a.C + m;  // class index == input pixel index
                    } else {
                        const int n = pp / (PH * PW), rem = pp - n * (PH * PW);
                        const int r = rem / PW;
                        const int iy = r * a.stride + ph, ix = (rem - r * PW) * a.stride + pw;
                        o = (((int64_t)n * a.H + iy) * a.W + ix) * a.C + m;
                    }
                    float g = v[j];
                    if (a.addsrc) g += __bfloat162float(a.addsrc[s * a.addsrc_stride_s + o]);
                    if (a.mask && !(__bfloat162float(a.mask[s * a.mask_stride_s + o]) > 0.0f)) g = 0.0f;
                    part += g;
                    outs[o] = __float2bfloat16_rn(g);
                }
            }
        }
        if (MODE == 1 && a.bpart && mvalid) {
            const int ptiles = (npix + 255) / 256;
            a.bpart[s * a.bpart_stride_s + ((int64_t)(cls * ptiles + blockIdx.y) * 2 + h) * a.C + m] = part;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kProdWarps) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

int conv_dgrad_parts(const ConvTcArgs& a) {
    const int npix = a.B * (a.H / a.stride) * (a.W / a.stride);
    return a.stride * a.stride * ((npix + 255) / 256) * 2;
}

void launch_conv_tc_fwd(const CUtensorMap& wmap, const CUtensorMap& bmap, const ConvTcArgs& a, int S,
                        cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(conv_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, cv::kSmem);
        attr = true;
    }
    const int npix = a.B * a.OH * a.OW;
    dim3 grid((a.CO + 127) / 128, (npix + 255) / 256, S);
    conv_tc_kernel<0><<<grid, cv::kThreads, cv::kSmem, st>>>(wmap, bmap, a);
}

void launch_conv_tc_dgrad(const CUtensorMap& wmapT, const CUtensorMap& bmap, const ConvTcArgs& a, int S,
                          cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(conv_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cv::kSmem);
        attr = true;
    }
    const int npix = a.B * (a.H / a.stride) * (a.W / a.stride);
    dim3 grid((a.C + 127) / 128, (npix + 255) / 256, S * a.stride * a.stride);
    conv_tc_kernel<1><<<grid, cv::kThreads, cv::kSmem, st>>>(wmapT, bmap, a);
}

// ============================================================================ wgrad
namespace cw {
constexpr int kEpiWarps = 8;
constexpr int kGatherWarps = 4;
constexpr int kThreads = (kEpiWarps + kGatherWarps + 2) * 32;
constexpr int kStages = 6;
constexpr int kAStage = 64 * 128 * 2;  // dYᵀ: 64 pixels × 128 co (two 64-wide MN blocks)
constexpr int kBStage = 64 * 64 * 2;   // X window: 64 pixels × 64 ci
constexpr int kSmem = 1024 + kStages * (kAStage + kBStage) + 256;
}  // namespace cw

__global__ void __launch_bounds__(cw::kThreads, 1)
    conv_wgrad_tc_kernel(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap xmap,
                         const ConvWgradArgs a) {
    using namespace cw;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const SampledLayer& L = a.L;
    const int taps = a.k * a.k;
    const int ci_tiles = a.C / 64;
    const int co_tiles = (a.CO + 127) / 128;
    int t = blockIdx.x;
    const int split = t % a.nsplit;
    t /= a.nsplit;
    const int cit = t % ci_tiles;
    t /= ci_tiles;
    const int tap = t % taps;
    const int cot = t / taps;
    const int co0 = cot * 128, ci0 = cit * 64, kh = tap / a.k, kw = tap % a.k;
    const int npix = a.B * a.OH * a.OW;
    const int nblk_all = (npix + 63) / 64;
    const int per = (nblk_all + a.nsplit - 1) / a.nsplit;
    const int blk0 = split * per, blk1 = min(nblk_all, blk0 + per);
    const int nblk = max(0, blk1 - blk0);
    const int S = a.S;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], a.tma_b ? 1 : kGatherWarps * 32 + 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps);
        }
        mbar_fence_init();
    }
    if (warp == kEpiWarps + kGatherWarps + 1) tmem_alloc(tslot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == kEpiWarps + kGatherWarps) {
        // ------------------------------------------------ TMA: dYᵀ blocks
        if (lane == 0 && nblk > 0) {
            tma_prefetch_desc(&gmap);
            if (a.tma_b) tma_prefetch_desc(&xmap);
            int it = 0;
            for (int s = 0; s < S; ++s)
                for (int b = 0; b < nblk; ++b, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_sleep(&empty[st], ph ^ 1);
                    mbar_arrive_expect_tx(&full[st], kAStage + (a.tma_b ? kBStage : 0));
                    uint8_t* dst = sA + st * kAStage;
                    const int pix0 = (blk0 + b) * 64;
                    tma_load_3d(&gmap, &full[st], dst, co0, pix0, s);
                    tma_load_3d(&gmap, &full[st], dst + 8192, co0 + 64, pix0, s);
                    if (a.tma_b) {  // stride 1: the shifted input window of these 64 pixels
                        const int n0 = pix0 / (a.OH * a.OW), y0 = (pix0 - n0 * a.OH * a.OW) / a.OW;
                        tma_load_5d(&xmap, &full[st], sB + st * kBStage, ci0, kw - a.pad, y0 + kh - a.pad,
                                    n0, a.X_stride_s == 0 ? 0 : s);
                    }
                }
        }
        __syncwarp();
    } else if (warp == kEpiWarps + kGatherWarps + 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0 && nblk > 0) {
            const uint32_t idesc = idesc_bf16(128, 64, 1, 1);
            int it = 0;
            for (int s = 0; s < S; ++s) {
                const int buf = s & 1;
                mbar_wait_sleep(&tempty[buf], ((s >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int b = 0; b < nblk; ++b, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_sleep(&full[st], ph);
                    fence_proxy_async_smem();
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + st * kAStage);
                    const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = sdesc_sw128(aBase + 2048 * q, 8192, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 2048 * q, 8192, 1024);
                        mma_bf16(tmem + buf * 64, ad, bd, idesc, (b | q) != 0 ? 1u : 0u);
                        mma_bf16(tmem + 128, ad, bd, idesc, (s | b | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else if (warp >= kEpiWarps) {
        // ------------------------------------------------ gather X windows: 64 rows × 8 chunks
        const int gt = threadIdx.x - kEpiWarps * 32;  // 0..127
        int it = 0;
        for (int s = 0; s < (a.tma_b ? 0 : S); ++s) {
            const __nv_bfloat16* xs = a.X + s * a.X_stride_s;
            for (int b = 0; b < nblk; ++b, ++it) {
                const int st = it % kStages;
                const uint32_t ph = (it / kStages) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                const uint32_t base = smem_u32(sB + st * kBStage);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = u * 128 + gt;  // 512 chunks
                    const int r = idx >> 3, j = idx & 7;
                    const int pix = (blk0 + b) * 64 + r;
                    const __nv_bfloat16* g = xs;
                    uint32_t bytes = 0;
                    if (pix < npix) {
                        const int n = pix / (a.OH * a.OW), rem = pix % (a.OH * a.OW);
                        const int iy = (rem / a.OW) * a.stride + kh - a.pad;
                        const int ix = (rem % a.OW) * a.stride + kw - a.pad;
                        if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
                            g = xs + (((int64_t)n * a.H + iy) * a.W + ix) * a.C_pad + ci0 + 8 * j;
                            bytes = 16;
                        }
                    }
                    cp_async16(base + r * 128 + ((j ^ (r & 7)) << 4), g, bytes);
                }
                cp_async_mbar_arrive(&full[st]);
            }
        }
    } else {
        // ------------------------------------------------ epilogue: ε regeneration + accumulation
        const int q = warp & 3, h = warp >> 2;
        const int co = co0 + 32 * q + lane;
        const int col = tap * a.C + ci0 + 32 * h;  // parameter column of this thread's first value
        const int Kt = taps * a.C;
        float ar[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) ar[j] = 0.0f;
        for (int s = 0; s < S && nblk > 0; ++s) {
            const int buf = s & 1;
            mbar_wait(&tfull[buf], (s >> 1) & 1);
            tc_fence_after();
            float d[32];
            __syncwarp();
            tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 64 + 32 * h, d);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if (co < a.CO) {
                const uint32_t sgw = (L.t_w << 20) | (a.kk.s0 + s);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint4 y = philox10(make_uint4((uint32_t)((col >> 2) + g), (uint32_t)co, sgw, a.kk.step),
                                             a.kk.key);
                    const float R0 = bm_radius(y.x);
                    const float2 cs0 = bm_sincos(y.y);
                    const float R1 = bm_radius(y.z);
                    const float2 cs1 = bm_sincos(y.w);
                    ar[4 * g + 0] = fmaf(d[4 * g + 0], __fmul_rn(R0, cs0.x), ar[4 * g + 0]);
                    ar[4 * g + 1] = fmaf(d[4 * g + 1], __fmul_rn(R0, cs0.y), ar[4 * g + 1]);
                    ar[4 * g + 2] = fmaf(d[4 * g + 2], __fmul_rn(R1, cs1.x), ar[4 * g + 2]);
                    ar[4 * g + 3] = fmaf(d[4 * g + 3], __fmul_rn(R1, cs1.y), ar[4 * g + 3]);
                }
            }
        }
        float am[32];
        __syncwarp();
        if (nblk > 0) {
            tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + 128 + 32 * h, am);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) am[j] = 0.0f;
        }
        if (co < a.CO) {
            const int64_t n = (int64_t)a.CO * Kt;
            float* pm = a.part + (int64_t)split * 2 * n + (int64_t)co * Kt + col;
            float* pr = pm + n;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                reinterpret_cast<float4*>(pm)[g] =
                    make_float4(a.scale * am[4 * g], a.scale * am[4 * g + 1], a.scale * am[4 * g + 2],
                                a.scale * am[4 * g + 3]);
                reinterpret_cast<float4*>(pr)[g] =
                    make_float4(a.scale * ar[4 * g], a.scale * ar[4 * g + 1], a.scale * ar[4 * g + 2],
                                a.scale * ar[4 * g + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + kGatherWarps + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

void launch_conv_tc_wgrad(const CUtensorMap& gmap, const CUtensorMap& xmap, const ConvWgradArgs& a,
                          cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(conv_wgrad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cw::kSmem);
        attr = true;
    }
    const int tiles = ((a.CO + 127) / 128) * a.k * a.k * (a.C / 64) * a.nsplit;
    conv_wgrad_tc_kernel<<<tiles, cw::kThreads, cw::kSmem, st>>>(gmap, xmap, a);
}

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

void launch_wgrad_split_reduce(const float* part, int nsplit, int64_t n, int64_t off, float* acc_mu,
                               float* acc_rho, cudaStream_t st) {
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
