// kernels_conv2.cu — persistent swap-AB tcgen05 implicit-GEMM convolution (K3 fwd, K4 dgrad).
//
//   fwd   D[pixel][co] = Σ_{kh,kw,ci} X[pixel ⊕ (kh,kw)][ci] · W_s[co][kh,kw,ci]
//   dgrad D[pixel][ci] = Σ_{kh,kw,co} dY[pixel ⊖ (kh,kw)][co] · W_s[co][kh,kw,ci]
//
// M = 128 pixels (TMEM lanes), N = up to 256 channels (TMEM columns), K = 64 per stage.
// Putting pixels on M makes every TMEM lane one NHWC row, so the epilogue reads 32
// consecutive channels per tcgen05.ld and moves them with 16-byte vector loads/stores, with
// bias, residual, ReLU, the ReLU mask of the layer input and the producer's bias-gradient
// partials fused. A operand: the activation (fwd) or dY (dgrad) window — 5-D TMA with OOB
// zero fill for stride-1 convs, a cp.async gather for stride 2 and the 3-channel stem. B
// operand: the W_s scratch (K-major for fwd, MN-major for dgrad) by TMA. Persistent CTAs
// walk a static tile schedule; two TMEM accumulators let tile i's epilogue overlap tile
// i+1's main loop.
#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_conv.cuh"
#include "tc_ptx.cuh"

namespace bnn {

// The MMA issuers fence the async proxy after a stage fills only when gather warps wrote it with
// generic-proxy stores; TMA-filled stages need no fence (-DBNN_ALWAYS_PROXY_FENCE restores it).
#ifdef BNN_ALWAYS_PROXY_FENCE
constexpr bool kAlwaysFence = true;
#else
constexpr bool kAlwaysFence = false;
#endif

using namespace ptx;

// pipeline depth cap (BNN_CONV_STAGES, default 4; ≤ 12), passed as a launch argument
static int conv_stage_cap() {
    static int cap = [] {
        const char* e = getenv("BNN_CONV_STAGES");
        const int v = e ? atoi(e) : 4;
        return v < 2 ? 2 : (v > 12 ? 12 : v);
    }();
    return cap;
}

static int conv_debug() {  // BNN_CONV_DEBUG: 1 = skip MMAs, 2 = skip operand loads (timing experiments)
    static int v = [] {
        const char* e = getenv("BNN_CONV_DEBUG");
        return e ? atoi(e) : 0;
    }();
    return v;
}

namespace c2 {
constexpr int kEpiWarps = 4;
constexpr int kGatherWarps = 4;
constexpr int kThreads = (kEpiWarps + kGatherWarps + 2) * 32;
constexpr int kAStage = 128 * 64 * 2;  // 16 KB pixel window
constexpr int kData = 216 * 1024;      // stages: as many (A 16 KB + B n_tile·128 B) as fit
constexpr int kSmem = 1024 + kData + 512 + 1024;
}  // namespace c2

__host__ __device__ __forceinline__ int floor_div(int a, int b) {  // b > 0
    const int q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

struct TileGeo {
    int s, cls, ptile, ntile;
};

template <int MODE>
__device__ __forceinline__ TileGeo tile_of(int t, int ntiles, int ptiles, int ncls) {
    TileGeo g;
    g.ntile = t % ntiles;
    t /= ntiles;
    g.ptile = t % ptiles;
    t /= ptiles;
    g.cls = t % ncls;
    g.s = t / ncls;
    return g;
}

// transpose-reduce: lane j ends with Σ over the warp's 32 lanes of v[j]
__device__ __forceinline__ float warp_transpose_sum(float* v, int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = upper ? v[i] : v[i + off];
            const float keep = upper ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// ReLU bitmask of 32 packed bf16 (4 × uint4, channel order): bit j = (channel j > 0)
__device__ __forceinline__ uint32_t relu_bits32(const uint4* w) {
    uint32_t bits = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t w4[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t lo = w4[e] & 0xFFFFu, hi = w4[e] >> 16;
            bits |= (uint32_t)((lo & 0x7FFFu) != 0 && (lo & 0x8000u) == 0) << (8 * q + 2 * e);
            bits |= (uint32_t)((hi & 0x7FFFu) != 0 && (hi & 0x8000u) == 0) << (8 * q + 2 * e + 1);
        }
    }
    return bits;
}

// Epilogue of one NHWC row segment: this thread's pixel (row offset `rowoff`, valid `pv`) and the
// 32 channels ch0 … ch0+31 in v (fp32 accumulators). fwd: + sampled bias, + residual, ReLU,
// RN-bf16 store. dgrad: + the other contribution, ReLU mask of the layer input, RN-bf16 store;
// v keeps the masked fp32 values (zero for invalid pixels) for the bias-gradient partials.
template <int MODE, bool BIAS = true>
__device__ __forceinline__ void epi_row32(const Conv2Args& a, float* v, bool pv, int64_t rowoff, int64_t so,
                                          int s, int ch0) {
    if (MODE == 0) {
        if (BIAS) {
        const float4* bs = reinterpret_cast<const float4*>(a.bias + (int64_t)s * a.CO + ch0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 b4 = __ldg(bs + q);
            v[4 * q] += b4.x;
            v[4 * q + 1] += b4.y;
            v[4 * q + 2] += b4.z;
            v[4 * q + 3] += b4.w;
        }
        }
        if (!pv) return;
        if (a.res) {
            const uint4* rp = reinterpret_cast<const uint4*>(a.res + so + rowoff + ch0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 r4 = __ldg(rp + q);
                const uint32_t w4[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    v[8 * q + 2 * e] += __uint_as_float(w4[e] << 16);
                    v[8 * q + 2 * e + 1] += __uint_as_float(w4[e] & 0xFFFF0000u);
                }
            }
        }
        uint4* op = reinterpret_cast<uint4*>(a.out + so + rowoff + ch0);
        uint4 pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float z[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) z[e] = a.relu ? fmaxf(v[8 * q + e], 0.0f) : v[8 * q + e];
            pk[q] = make_uint4(pack_bf16x2(z[0], z[1]), pack_bf16x2(z[2], z[3]), pack_bf16x2(z[4], z[5]),
                               pack_bf16x2(z[6], z[7]));
            op[q] = pk[q];
        }
        if (a.mbits_out) a.mbits_out[(so + rowoff + ch0) >> 5] = relu_bits32(pk);
    } else {
        if (!pv) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.0f;
            return;
        }
        if (a.addsrc) {
            const uint4* ap = reinterpret_cast<const uint4*>(a.addsrc + so + rowoff + ch0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 r4 = ap[q];
                const uint32_t w4[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    v[8 * q + 2 * e] += __uint_as_float(w4[e] << 16);
                    v[8 * q + 2 * e + 1] += __uint_as_float(w4[e] & 0xFFFF0000u);
                }
            }
        }
        if (a.mbits) {
            const uint32_t mb = __ldg(a.mbits + ((so + rowoff + ch0) >> 5));
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (!((mb >> j) & 1u)) v[j] = 0.0f;
        } else if (a.mask) {
            const uint4* mp = reinterpret_cast<const uint4*>(a.mask + so + rowoff + ch0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 m4 = __ldg(mp + q);
                const uint32_t w4[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (!(__uint_as_float(w4[e] << 16) > 0.0f)) v[8 * q + 2 * e] = 0.0f;
                    if (!(__uint_as_float(w4[e] & 0xFFFF0000u) > 0.0f)) v[8 * q + 2 * e + 1] = 0.0f;
                }
            }
        }
        uint4* op = reinterpret_cast<uint4*>(a.out + so + rowoff + ch0);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            op[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                               pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
    }
}

// epi_row32 with the residual (fwd) / other contribution + mask (dgrad) rows already loaded
// (x1, x2: 32 bf16 each) and the bias already added.
template <int MODE>
__device__ __forceinline__ void epi_apply32(const Conv2Args& a, float* v, bool pv, int64_t rowoff, int64_t so,
                                            int ch0, const uint4* x1, uint32_t mb) {
    if (!pv) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        return;
    }
    const bool add = MODE == 0 ? a.res != nullptr : a.addsrc != nullptr;
    if (add) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t w4[4] = {x1[q].x, x1[q].y, x1[q].z, x1[q].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[8 * q + 2 * e] += __uint_as_float(w4[e] << 16);
                v[8 * q + 2 * e + 1] += __uint_as_float(w4[e] & 0xFFFF0000u);
            }
        }
    }
    if (MODE == 0) {
        if (a.relu) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
        }
    } else if (a.mbits) {  // mb = the input's ReLU bitmask word
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (!((mb >> j) & 1u)) v[j] = 0.0f;
    }
    uint4* op = reinterpret_cast<uint4*>(a.out + so + rowoff + ch0);
    uint4 pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        pk[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                           pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        op[q] = pk[q];
    }
    if (MODE == 0 && a.mbits_out) a.mbits_out[(so + rowoff + ch0) >> 5] = relu_bits32(pk);
}

// CPS CTAs per SM: 1 (216 KB of stages, two TMEM accumulators) or 2 (96 KB, one accumulator each:
// two MMA issue streams per SM, and a 256-tile stage-4 layer fits one wave of 296 slots)
template <int MODE, int CPS>
__global__ void __launch_bounds__(c2::kThreads, CPS)
    conv2_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap wmap,
                 const Conv2Args a, const int g_max_stages_arg) {
    using namespace c2;
    constexpr int NB = CPS == 1 ? 2 : 1;
    constexpr int DATA = CPS == 1 ? kData : 96 * 1024;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment as an offset into the __shared__ array: the pointer keeps the shared
    // address space, so plain loads/stores through it compile to LDS/STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    const int kBStage = a.n_tile * 128;
    const int kStages = min(g_max_stages_arg, DATA / (kAStage + kBStage));
    uint8_t* sB = smem + kStages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
    int* staps = reinterpret_cast<int*>(tslot + 4);  // [4 classes][9 taps] + counts
    float* bred = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);  // [2][4 warps][32]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncls = MODE == 1 ? a.stride * a.stride : 1;
    const int PH = MODE == 0 ? a.OH : a.H / a.stride, PW = MODE == 0 ? a.OW : a.W / a.stride;
    const int P = a.B * PH * PW;
    const int ptiles = (P + 127) / 128;
    const int Ntot = MODE == 0 ? a.CO : a.C;
    const int ntiles = (Ntot + a.n_tile - 1) / a.n_tile;
    const int T = a.S * ncls * ptiles * ntiles;
    const int cblocks = (a.CO + 63) / 64;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1 + (a.tma_a ? 0 : kGatherWarps * 32));
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps);
        }
        mbar_fence_init();
        // valid taps per parity class (dgrad): staps[cls*10 + 9] = count
        for (int cl = 0; cl < ncls; ++cl) {
            const int ph = cl / a.stride, pw = cl % a.stride;
            int cnt = 0;
            if (MODE == 1) {
                for (int kh = 0; kh < a.k; ++kh)
                    for (int kw = 0; kw < a.k; ++kw)
                        if ((ph + a.pad - kh) % a.stride == 0 && (pw + a.pad - kw) % a.stride == 0)
                            staps[cl * 10 + cnt++] = kh * a.k + kw;
            }
            staps[cl * 10 + 9] = cnt;
        }
    }
    if (warp == kEpiWarps + kGatherWarps + 1) tmem_alloc(tslot, NB * 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    auto nkb_of = [&](int cls) { return MODE == 0 ? a.K_pad / 64 : staps[cls * 10 + 9] * cblocks; };

    if (warp == kEpiWarps + kGatherWarps) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&wmap);
            if (a.tma_a) tma_prefetch_desc(&amap);
            const int cpb = a.C_pad >> 6;
            const uint32_t bbytes = (uint32_t)a.n_tile * 128;
            int it = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const TileGeo g = tile_of<MODE>(t, ntiles, ptiles, ncls);
                const int p0 = g.ptile * 128, n0 = g.ntile * a.n_tile;
                const int img0 = p0 / (PH * PW), y0 = (p0 - img0 * PH * PW) / PW;
                const int nkb = nkb_of(g.cls);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_role(&empty[st], ph ^ 1);
                    if (a.dbg & 2) {  // feed-rate experiment: no loads
                        mbar_arrive_expect_tx(&full[st], 0);
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[st], bbytes + (a.tma_a ? kAStage : 0));
                    uint8_t* dA = sA + st * kAStage;
                    uint8_t* dB = sB + st * kBStage;
                    if (MODE == 0) {
                        tma_load_3d(&wmap, &full[st], dB, kb * 64, n0, g.s);
                        if (a.tma_a) {
                            const int tap = kb / cpb, c0 = (kb - tap * cpb) * 64;
                            const int kh = tap / a.k, kw = tap - kh * a.k;
                            // stride s: the map traverses W and H with element stride s
                            tma_load_5d(&amap, &full[st], dA, c0, kw - a.pad, a.stride * y0 + kh - a.pad, img0,
                                        a.src_stride_s == 0 ? 0 : g.s);
                        }
                    } else {
                        const int ti = kb / cblocks, tap = staps[g.cls * 10 + ti], cb = kb - ti * cblocks;
                        // W_sᵀ: n_tile/64 channel blocks of 64 ci × 64 co in ONE op (5-D map, box 64×1×64×nb×1)
                        tma_load_5d(&wmap, &full[st], dB, 0, tap, cb * 64, n0 / 64, g.s);
                        if (a.tma_a) {
                            const int kh = tap / a.k, kw = tap - kh * a.k;
                            // dY window of this parity class: input pixel (s·y'+ph, s·x'+pw) takes
                            // dY(y' + (ph+pad-kh)/s, x' + (pw+pad-kw)/s) — a plain shifted window
                            const int ph = g.cls / a.stride, pw = g.cls - (g.cls / a.stride) * a.stride;
                            tma_load_5d(&amap, &full[st], dA, cb * 64, (pw + a.pad - kw) / a.stride,
                                        y0 + (ph + a.pad - kh) / a.stride, img0, g.s);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == kEpiWarps + kGatherWarps + 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, a.n_tile, 0, MODE == 1 ? 1 : 0);
            int it = 0, tl = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
                const TileGeo g = tile_of<MODE>(t, ntiles, ptiles, ncls);
                const int buf = tl % NB;
                mbar_wait_role(&tempty[buf], ((tl / NB) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                const int nkb = nkb_of(g.cls);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_role(&full[st], ph);
                    if (kAlwaysFence || !(a.tma_a)) fence_proxy_async_smem();  // gathered (generic-proxy) operands only
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + st * kAStage);
                    const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = sdesc_sw128(aBase + 32 * q, 16, 1024);
                        const uint64_t bd = MODE == 0 ? sdesc_sw128(bBase + 32 * q, 16, 1024)
                                                      : sdesc_sw128(bBase + 2048 * q, 8192, 1024);
                        if (!(a.dbg & 1)) mma_bf16(d, ad, bd, idesc, (kb | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[buf]);  // no MMAs (empty parity class): arrives at once
            }
        }
        __syncwarp();
    } else if (warp >= kEpiWarps) {
        // ------------------------------------------------ gather producers (stride 2 / stem)
        if (!a.tma_a) {
            const int r = threadIdx.x - kEpiWarps * 32;  // pixel row 0..127
            const int cpb = a.C_pad >> 6;
            int it = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const TileGeo g = tile_of<MODE>(t, ntiles, ptiles, ncls);
                const int ph = g.cls / a.stride, pw = g.cls % a.stride;
                const int pix = g.ptile * 128 + r;
                const bool pv = pix < P;
                const int pn = pv ? pix / (PH * PW) : 0;
                const int rem = pv ? pix - pn * PH * PW : 0;
                const int py = MODE == 0 ? rem / PW : (rem / PW) * a.stride + ph;
                const int px = MODE == 0 ? rem % PW : (rem % PW) * a.stride + pw;
                const __nv_bfloat16* src = a.src + g.s * a.src_stride_s;
                const int nkb = nkb_of(g.cls);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kStages;
                    const uint32_t phs = (it / kStages) & 1;
                    gather_wait(&empty[st], phs ^ 1);
                    const uint32_t base = smem_u32(sA + st * kAStage) + r * 128;
                    if (MODE == 0 && cpb == 0) {  // stem: 8 taps × 8 channels per K block
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int tap = kb * 8 + j;
                            const int kh = tap / a.k, kw = tap - (tap / a.k) * a.k;
                            const int iy = py * a.stride + kh - a.pad, ix = px * a.stride + kw - a.pad;
                            const bool ok = pv && tap < a.k * a.k && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                            const __nv_bfloat16* gp = ok ? src + (((int64_t)pn * a.H + iy) * a.W + ix) * a.C_pad : src;
                            cp_async16(base + ((j ^ (r & 7)) << 4), gp, ok ? 16u : 0u);
                        }
                    } else {
                        int kh, kw, c0;
                        if (MODE == 0) {
                            const int tap = kb / cpb;
                            c0 = (kb - tap * cpb) * 64;
                            kh = tap / a.k;
                            kw = tap - kh * a.k;
                        } else {
                            const int ti = kb / cblocks, tap = staps[g.cls * 10 + ti];
                            c0 = (kb - ti * cblocks) * 64;
                            kh = tap / a.k;
                            kw = tap - kh * a.k;
                        }
                        bool ok;
                        const __nv_bfloat16* gp = src;
                        if (MODE == 0) {
                            const int iy = py * a.stride + kh - a.pad, ix = px * a.stride + kw - a.pad;
                            ok = pv && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                            if (ok) gp = src + (((int64_t)pn * a.H + iy) * a.W + ix) * a.C_pad + c0;
                        } else {
                            const int ty = py + a.pad - kh, tx = px + a.pad - kw;
                            const int oy = ty / a.stride, ox = tx / a.stride;
                            ok = pv && ty >= 0 && tx >= 0 && oy < a.OH && ox < a.OW;
                            if (ok) gp = src + (((int64_t)pn * a.OH + oy) * a.OW + ox) * a.CO + c0;
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            cp_async16(base + ((j ^ (r & 7)) << 4), gp + 8 * j, ok ? 16u : 0u);
                    }
                    cp_async_mbar_arrive(&full[st]);
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue: thread = pixel row
        const int row = 32 * warp + lane;
        int tl = 0, nred = 0;
        for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
            const TileGeo g = tile_of<MODE>(t, ntiles, ptiles, ncls);
            const int buf = tl % NB;
            const int nkb = nkb_of(g.cls);
            epi_wait(&tfull[buf], (tl / NB) & 1);
            tc_fence_after();
            const int pix = g.ptile * 128 + row;
            const bool pv = pix < P;
            int64_t rowoff = 0;  // element offset of this pixel's channel 0
            if (pv) {
                if (MODE == 0 || a.stride == 1) {
                    rowoff = (int64_t)pix * Ntot;
                } else {
                    const int ph = g.cls / a.stride, pw = g.cls % a.stride;
                    const int pn = pix / (PH * PW), rem = pix - pn * PH * PW;
                    const int iy = (rem / PW) * a.stride + ph, ix = (rem % PW) * a.stride + pw;
                    rowoff = (((int64_t)pn * a.H + iy) * a.W + ix) * a.C;
                }
            }
            const int n0 = g.ntile * a.n_tile;
            const int64_t so = (int64_t)g.s * a.out_stride_s;
            for (int c = 0; c < a.n_tile / 32; ++c) {
                float v[32];
                __syncwarp();
                if (nkb > 0) {
                    tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + buf * 256 + c * 32, v);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.0f;
                }
                const int ch0 = n0 + c * 32;
                epi_row32<MODE>(a, v, pv, rowoff, so, g.s, ch0);
                if (MODE == 1) {
                    if (a.bpart) {  // fp32 bias partials (pre-rounding) over the tile's 128 pixels
                        float* red = bred + (nred++ & 1) * 128;
                        red[warp * 32 + lane] = warp_transpose_sum(v, lane);
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (warp == 0)
                            a.bpart[(int64_t)g.s * a.bpart_stride_s + (int64_t)(g.cls * ptiles + g.ptile) * a.C +
                                    ch0 + lane] = (red[lane] + red[32 + lane]) + (red[64 + lane] + red[96 + lane]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + kGatherWarps + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, NB * 256);
    }
}

// CTAs per SM of the swap-AB conv: 2 for the data gradient (C3 stage 4: 91–96 → 77–83 µs, stage 3
// 96–101 → 90–100), 1 for the forward (stage 4: 82 → 90 µs with two); BNN_CONV2_CPS=1|2 forces both
static int conv2_cps(int mode) {
    static int v = [] {
        const char* e = getenv("BNN_CONV2_CPS");
        const int x = e ? atoi(e) : 0;
        return x == 1 || x == 2 ? x : 0;
    }();
    return v ? v : (mode == 1 ? 2 : 1);
}

int conv2_dgrad_parts(const Conv2Args& a) {
    const int P = a.B * (a.H / a.stride) * (a.W / a.stride);
    return a.stride * a.stride * ((P + 127) / 128);
}

template <int MODE>
static void launch_conv2(const CUtensorMap& amap, const CUtensorMap& wmap, const Conv2Args& a,
                         cudaStream_t st) {
    const int ncls = MODE == 1 ? a.stride * a.stride : 1;
    const int PH = MODE == 0 ? a.OH : a.H / a.stride, PW = MODE == 0 ? a.OW : a.W / a.stride;
    const int P = a.B * PH * PW;
    const int Ntot = MODE == 0 ? a.CO : a.C;
    const int T = a.S * ncls * ((P + 127) / 128) * ((Ntot + a.n_tile - 1) / a.n_tile);
    Conv2Args b = a;
    b.dbg = conv_debug();
    if (conv2_cps(MODE) == 2) {
        constexpr int smem = 1024 + 96 * 1024 + 512 + 1024;
        ensure_smem_attr(reinterpret_cast<const void*>(conv2_kernel<MODE, 2>), smem);
        conv2_kernel<MODE, 2><<<std::min(T, 2 * kNumSMs), c2::kThreads, smem, st>>>(amap, wmap, b, conv_stage_cap());
        return;
    }
    ensure_smem_attr(reinterpret_cast<const void*>(conv2_kernel<MODE, 1>), c2::kSmem);
    conv2_kernel<MODE, 1><<<std::min(T, kNumSMs), c2::kThreads, c2::kSmem, st>>>(amap, wmap, b, conv_stage_cap());
}

void launch_conv2_fwd(const CUtensorMap& amap, const CUtensorMap& wmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv2<0>(amap, wmap, a, st);
}
void launch_conv2_dgrad(const CUtensorMap& amap, const CUtensorMap& wmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv2<1>(amap, wmap, a, st);
}

// ============================================================================ conv3 (channels on M)
// For layers whose output channel count (fwd: CO, dgrad: C) is ≤ 128 the swap-AB tile would run
// tcgen05.mma at N = 64/128 — and an M=128 MMA costs the same ~130 cycles per K=16 for any
// N ≤ 256 (scripts/mma_bench.cu, profiles/r01). Here M = 128 channels (weights, the A operand)
// and N = 256 pixels (activation / dY window, the B operand); the epilogue transposes each
// warp's 32 channels × 32 pixels through shared memory so the NHWC row epilogue is reused.
namespace c3 {
constexpr int kEpiWarps = 8;
constexpr int kGatherWarps = 4;
constexpr int kThreads = (kEpiWarps + kGatherWarps + 2) * 32;
// HALO variant: no gather warps (every operand arrives by TMA); 8 epilogue warps, 3 A stages,
// two window stages, two 256-column TMEM accumulators, one CTA per SM. (Measured and reverted,
// round 2: 16 epilogue warps, and two CTAs per SM with one window / accumulator each — both
// slower; a thread = channel epilogue without the shared-memory transpose — 1.8× slower.)
constexpr int kEpiWarpsH = 8;
constexpr int kThreadsH = (kEpiWarpsH + 2) * 32;
constexpr int kTransPitch = 33;  // floats per transposed row (conflict-free scalar stores and loads)
constexpr int kStages = 3;  // pipeline depth is not the limiter (BNN_CONV_STAGES sweep, profiles/r01)
constexpr int kAStage = 128 * 64 * 2;  // 16 KB weights (128 channel rows)
constexpr int kBStage = 256 * 64 * 2;  // 32 KB pixel window (256 rows)
constexpr int kTrans = kEpiWarps * 32 * kTransPitch * 4;
constexpr int kTransH = kEpiWarpsH * 32 * kTransPitch * 4;
constexpr int kWin = kStages * kBStage / 2;  // HALO: two window stages in the B-stage region (48 KB each)
constexpr int kStagesH = 3;                  // HALO: A stages
constexpr int kSmem = 1024 + kStages * (kAStage + kBStage) + kTrans + 512 + 2048;
constexpr int kSmemH = 1024 + kStagesH * kAStage + 2 * kWin + kTransH + 512 + 2 * kEpiWarpsH * 32 * 4;
static_assert(kSmemH <= 227 * 1024, "conv3 halo shared memory");
static_assert(kSmem <= 227 * 1024, "conv3 shared memory");
}  // namespace c3

// HALO (stride-1 3×3 convs with 64 input channels of the B operand): tiles are 256
// consecutive pixels of the padded pixel stream — per image (H + 1) rows (the last one a zero
// separator shared by neighbouring images) × (W + 2) columns (zero columns at both ends) — and
// the CTA loads ONE window of whole padded rows around the tile per tile (≤ kWin bytes, one
// 1-row TMA box per padded row with OOB zero fill). Every tap's B operand is the window at a
// row offset dh·(W+2) + dw: SWIZZLE_128B is a function of the shared address, so a descriptor
// may start at any 128-B row (scripts/halo_desc_test.cu, profiles/r02/halo_desc_test.txt).
// L2→SM traffic per tile: one ≈ 48 KB window instead of nine 32 KB tap windows; the padded
// rows / columns cost (H+1)(W+2)/(HW) − 1 = 9.6 % more MMA columns at 32×32.
template <int MODE, bool HALO>
__global__ void __launch_bounds__(HALO ? c3::kThreadsH : c3::kThreads, 1)
    conv3_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap bmap,
                 const Conv2Args a) {
    using namespace c3;
    // HALO: the B stages become two window stages, so the 16 KB A (weight) stages can be deeper:
    // the A loads are L2 hits but ~1–2 µs in flight, against ≈ 0.3 µs of MMAs per k-block
    constexpr int NST = HALO ? kStagesH : kStages;
    constexpr int NEPI = HALO ? kEpiWarpsH : kEpiWarps;     // epilogue warps 0 … NEPI-1
    constexpr int NGATH = HALO ? 0 : kGatherWarps;          // gather warps (stride-2 / stem operands)
    constexpr int WTMA = NEPI + NGATH, WMMA = WTMA + 1;     // the TMA and MMA warps
    constexpr int NBUF = 2;                                 // TMEM accumulators of 256 columns
    constexpr int NWIN = 2;                                 // HALO window stages
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment as an offset into the __shared__ array: the pointer keeps the shared
    // address space, so plain loads/stores through it compile to LDS/STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + NST * kAStage;
    float* trans = reinterpret_cast<float*>(sB + (HALO ? NWIN * kWin : kStages * kBStage));  // B stages / HALO window
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(trans) + (HALO ? kTransH : kTrans));
    uint64_t* full = bars;
    uint64_t* empty = bars + NST;
    uint64_t* tfull = bars + 2 * NST;
    uint64_t* tempty = bars + 2 * NST + 2;
    uint64_t* wfull = bars + 2 * NST + 4;   // HALO: window stages (the sB region, 2 × kWin)
    uint64_t* wempty = bars + 2 * NST + 6;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 8);
    int* staps = reinterpret_cast<int*>(tslot + 4);  // [4 classes][9 taps] + counts
    float* bred = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);  // [2][8 warps][32]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncls = MODE == 1 ? a.stride * a.stride : 1;
    const int PH = MODE == 0 ? a.OH : a.H / a.stride, PW = MODE == 0 ? a.OW : a.W / a.stride;
    const int P = a.B * PH * PW;
    // padded stream (HALO): PWp columns per row, PH + 1 rows per image
    const int PWp = PW + 2, PHp = PH + 1;
    const int ptiles = HALO ? (a.B * PHp * PWp + 255) / 256 : (P + 255) / 256;
    // 64-channel layers: TMEM rows 64-127 repeat rows 0-63 (the A tile is loaded twice), so all
    // eight epilogue warps have channels to work on (MMA cost is the same for any M ≤ 128)
    const bool dup = (MODE == 0 ? a.CO : a.C) <= 64;
    const int Mtot = MODE == 0 ? a.CO : a.C;
    const int mtiles = (Mtot + 127) / 128;
    const int T = a.S * ncls * ptiles * mtiles;
    const int cblocks = (a.CO + 63) / 64;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1 + (a.tma_a ? 0 : NGATH * 32));
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], NEPI);
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 1);
        }
        mbar_fence_init();
        for (int cl = 0; cl < ncls; ++cl) {
            const int ph = cl / a.stride, pw = cl % a.stride;
            int cnt = 0;
            if (MODE == 1) {
                for (int kh = 0; kh < a.k; ++kh)
                    for (int kw = 0; kw < a.k; ++kw)
                        if ((ph + a.pad - kh) % a.stride == 0 && (pw + a.pad - kw) % a.stride == 0)
                            staps[cl * 10 + cnt++] = kh * a.k + kw;
            }
            staps[cl * 10 + 9] = cnt;
        }
    }
    if (warp == WMMA) tmem_alloc(tslot, NBUF * 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
#ifdef C3_PROF
    long long p_full = 0, p_tempty = 0, p_tfull = 0, p_empty = 0;
    const long long p_start = clock64();
#endif
    auto nkb_of = [&](int cls) { return MODE == 0 ? a.K_pad / 64 : staps[cls * 10 + 9] * cblocks; };

    if (warp == WTMA) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&wmap);
            if (a.tma_a) tma_prefetch_desc(&bmap);
            const int cpb = a.C_pad >> 6;
            int it = 0, tl = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
                const TileGeo g = tile_of<MODE>(t, mtiles, ptiles, ncls);
                const int p0 = g.ptile * 256, m0 = g.ntile * 128;
                const int img0 = p0 / (PH * PW), y0 = (p0 - img0 * PH * PW) / PW;
                const int nkb = nkb_of(g.cls);
                if (HALO) {  // the tile's window: padded rows rs … re, one TMA box per row
                    const int ws = tl % NWIN;
                    mbar_wait_role(&wempty[ws], ((tl / NWIN) & 1) ^ 1);
                    const int rs = floor_div(p0 - PWp - 1, PWp), re = floor_div(p0 + 256 + PWp, PWp);
                    uint8_t* win = sB + ws * kWin;
                    if (a.dbg & 2) {
                        mbar_arrive_expect_tx(&wfull[ws], 0);
                    } else {
                        mbar_arrive_expect_tx(&wfull[ws], (uint32_t)((re - rs + 1) * PWp * 128));
                        for (int r = rs; r <= re; ++r) {
                            const int b = floor_div(r, PHp), y = r - b * PHp;  // y == PH: separator (OOB: zeros)
                            tma_load_5d(&bmap, &wfull[ws], win + (r - rs) * PWp * 128, 0, -1, y, b,
                                        a.src_stride_s == 0 ? 0 : g.s);
                        }
                    }
                }
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % NST;
                    const uint32_t ph = (it / NST) & 1;
#ifdef C3_PROF
                    const long long q0 = clock64();
#endif
                    mbar_wait_role(&empty[st], ph ^ 1);
#ifdef C3_PROF
                    p_empty += clock64() - q0;
#endif
                    if (a.dbg & 2) {  // feed-rate experiment: no loads
                        mbar_arrive_expect_tx(&full[st], 0);
                        continue;
                    }
                    // A box: 128 weight rows, or 64 for a 64-channel layer (rows 64-127 then unused)
                    mbar_arrive_expect_tx(&full[st], kAStage + (a.tma_a && !HALO ? kBStage : 0));
                    uint8_t* dA = sA + st * kAStage;
                    uint8_t* dB = sB + st * kBStage;
                    if (MODE == 0) {
                        tma_load_3d(&wmap, &full[st], dA, kb * 64, m0, g.s);  // 128 rows, or 64 (dup)
                        if (dup) tma_load_3d(&wmap, &full[st], dA + 8192, kb * 64, m0, g.s);
                        if (a.tma_a && !HALO) {
                            const int tap = kb / cpb, c0 = (kb - tap * cpb) * 64;
                            const int kh = tap / a.k, kw = tap - kh * a.k;
                            tma_load_5d(&bmap, &full[st], dB, c0, kw - a.pad, a.stride * y0 + kh - a.pad, img0,
                                        a.src_stride_s == 0 ? 0 : g.s);
                        }
                    } else {
                        const int ti = kb / cblocks, tap = staps[g.cls * 10 + ti], cb = kb - ti * cblocks;
                        tma_load_5d(&wmap, &full[st], dA, 0, tap, cb * 64, m0 / 64, g.s);  // 2 ci blocks, or 1 (dup)
                        if (dup) tma_load_5d(&wmap, &full[st], dA + 8192, 0, tap, cb * 64, m0 / 64, g.s);
                        if (a.tma_a && !HALO) {
                            const int kh = tap / a.k, kw = tap - kh * a.k;
                            const int ph = g.cls / a.stride, pw = g.cls - (g.cls / a.stride) * a.stride;
                            tma_load_5d(&bmap, &full[st], dB, cb * 64, (pw + a.pad - kw) / a.stride,
                                        y0 + (ph + a.pad - kh) / a.stride, img0, g.s);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, 256, MODE == 1 ? 1 : 0, 0);
            int it = 0, tl = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
                const TileGeo g = tile_of<MODE>(t, mtiles, ptiles, ncls);
                const int buf = tl % NBUF;
#ifdef C3_PROF
                const long long q1 = clock64();
#endif
                mbar_wait_role(&tempty[buf], ((tl / NBUF) & 1) ^ 1);
#ifdef C3_PROF
                p_tempty += clock64() - q1;
#endif
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                const int nkb = nkb_of(g.cls);
                // HALO: row of the window where the tile's first pixel sits (tap (0, 0) offset)
                const int ws = tl % NWIN;
                const int wrow0 = HALO ? g.ptile * 256 - floor_div(g.ptile * 256 - PWp - 1, PWp) * PWp : 0;
                if (HALO) mbar_wait_role(&wfull[ws], (tl / NWIN) & 1);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % NST;
                    const uint32_t ph = (it / NST) & 1;
#ifdef C3_PROF
                    const long long q2 = clock64();
#endif
                    mbar_wait_role(&full[st], ph);
#ifdef C3_PROF
                    p_full += clock64() - q2;
#endif
                    if (kAlwaysFence || !(a.tma_a || HALO)) fence_proxy_async_smem();  // gathered (generic-proxy) operands only
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + st * kAStage);
                    uint32_t bBase = smem_u32(sB + st * kBStage);
                    if (HALO) {  // tap of this k-block (one 64-channel block per tap)
                        const int tap = MODE == 0 ? kb : staps[g.cls * 10 + kb];
                        const int kh = tap / 3, kw = tap - 3 * (tap / 3);
                        const int dh = MODE == 0 ? kh - 1 : 1 - kh, dw = MODE == 0 ? kw - 1 : 1 - kw;
                        bBase = smem_u32(sB + ws * kWin) + (uint32_t)(wrow0 + dh * PWp + dw) * 128u;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = MODE == 0 ? sdesc_sw128(aBase + 32 * q, 16, 1024)
                                                      : sdesc_sw128(aBase + 2048 * q, 8192, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 32 * q, 16, 1024);
                        if (!(a.dbg & 1)) mma_bf16(d, ad, bd, idesc, (kb | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                if (HALO) mma_commit(&wempty[ws]);  // the window is free once this tile's MMAs are done
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else if (warp >= NEPI) {
        // ------------------------------------------------ gather producers (stride 2 / stem): 256 rows
        if (!a.tma_a && !HALO) {
            const int gt = threadIdx.x - NEPI * 32;  // pixel rows gt and gt + 128
            const int cpb = a.C_pad >> 6;
            int it = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const TileGeo g = tile_of<MODE>(t, mtiles, ptiles, ncls);
                const int ph = g.cls / a.stride, pw = g.cls % a.stride;
                int py[2], px[2], pn[2];
                bool pv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pix = g.ptile * 256 + gt + 128 * h;
                    pv[h] = pix < P;
                    pn[h] = pv[h] ? pix / (PH * PW) : 0;
                    const int rem = pv[h] ? pix - pn[h] * PH * PW : 0;
                    py[h] = MODE == 0 ? rem / PW : (rem / PW) * a.stride + ph;
                    px[h] = MODE == 0 ? rem % PW : (rem % PW) * a.stride + pw;
                }
                const __nv_bfloat16* src = a.src + g.s * a.src_stride_s;
                const int nkb = nkb_of(g.cls);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % NST;
                    const uint32_t phs = (it / NST) & 1;
                    gather_wait(&empty[st], phs ^ 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = gt + 128 * h;
                        const uint32_t base = smem_u32(sB + st * kBStage) + r * 128;
                        if (MODE == 0 && cpb == 0) {  // stem: 8 taps × 8 channels per K block
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int tap = kb * 8 + j;
                                const int kh = tap / a.k, kw = tap - kh * a.k;
                                const int iy = py[h] * a.stride + kh - a.pad, ix = px[h] * a.stride + kw - a.pad;
                                const bool ok = pv[h] && tap < a.k * a.k && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                                const __nv_bfloat16* gp =
                                    ok ? src + (((int64_t)pn[h] * a.H + iy) * a.W + ix) * a.C_pad : src;
                                cp_async16(base + ((j ^ (r & 7)) << 4), gp, ok ? 16u : 0u);
                            }
                        } else {
                            int kh, kw, c0;
                            if (MODE == 0) {
                                const int tap = kb / cpb;
                                c0 = (kb - tap * cpb) * 64;
                                kh = tap / a.k;
                                kw = tap - kh * a.k;
                            } else {
                                const int ti = kb / cblocks, tap = staps[g.cls * 10 + ti];
                                c0 = (kb - ti * cblocks) * 64;
                                kh = tap / a.k;
                                kw = tap - kh * a.k;
                            }
                            bool ok;
                            const __nv_bfloat16* gp = src;
                            if (MODE == 0) {
                                const int iy = py[h] * a.stride + kh - a.pad, ix = px[h] * a.stride + kw - a.pad;
                                ok = pv[h] && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                                if (ok) gp = src + (((int64_t)pn[h] * a.H + iy) * a.W + ix) * a.C_pad + c0;
                            } else {
                                const int ty = py[h] + a.pad - kh, tx = px[h] + a.pad - kw;
                                const int oy = ty / a.stride, ox = tx / a.stride;
                                ok = pv[h] && ty >= 0 && tx >= 0 && oy < a.OH && ox < a.OW;
                                if (ok) gp = src + (((int64_t)pn[h] * a.OH + oy) * a.OW + ox) * a.CO + c0;
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                cp_async16(base + ((j ^ (r & 7)) << 4), gp + 8 * j, ok ? 16u : 0u);
                        }
                    }
                    cp_async_mbar_arrive(&full[st]);
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue: 8 warps; warp ↔ TMEM lane quadrant q = warp & 3
        // (32 channels), a subset of the tile's eight 32-pixel chunks; each chunk is transposed
        // through shared memory so the thread = pixel NHWC row epilogue (epi_row32) applies.
        // 64-channel layers (dup): quadrants 2,3 repeat channels 0-63, so all 8 warps work.
        float* tr = trans + warp * 32 * kTransPitch;
        const int q = warp & 3;
        const int cg = dup ? (q & 1) : q;                                   // channel group
        // the NEPI warps of each quadrant share its chunks: dup → 2·NEPI/8 warps per channel
        // group over 8 chunks (8 warps: 2 chunks each; 16 warps: 1), else NEPI/4 warps per group
        const int c_first = dup ? ((q >> 1) + 2 * (warp >> 2)) : (warp >> 2);  // first chunk
        const int c_step = dup ? NEPI / 2 : NEPI / 4;
        int tl = 0;
        for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
            const TileGeo g = tile_of<MODE>(t, mtiles, ptiles, ncls);
            const int buf = tl % NBUF;
            const int nkb = nkb_of(g.cls);
            const int ch0 = g.ntile * 128 + 32 * cg;
            const bool active = ch0 < Mtot;
            const int64_t so = (int64_t)g.s * a.out_stride_s;
            const float bias = (MODE == 0 && active) ? __ldg(a.bias + (int64_t)g.s * a.CO + ch0 + lane) : 0.0f;
            float bsum = 0.0f;
            // pixel row of chunk c for this lane (thread = pixel after the transpose)
            auto row_of = [&](int c, bool& pv) -> int64_t {
                const int pix = g.ptile * 256 + 32 * c + lane;
                if (HALO) {  // padded stream → (image, row, column); pad columns / separator rows invalid
                    const int r = pix / PWp, cx = pix - r * PWp, b = r / PHp, y = r - b * PHp;
                    pv = b < a.B && y < PH && cx >= 1 && cx <= PW;
                    return pv ? (((int64_t)b * PH + y) * PW + cx - 1) * Mtot : 0;
                }
                pv = pix < P;
                if (!pv) return 0;
                if (MODE == 0 || a.stride == 1) return (int64_t)pix * Mtot;
                const int ph = g.cls / a.stride, pw = g.cls % a.stride;
                const int pn = pix / (PH * PW), rem = pix - pn * PH * PW;
                const int iy = (rem / PW) * a.stride + ph, ix = (rem % PW) * a.stride + pw;
                return (((int64_t)pn * a.H + iy) * a.W + ix) * a.C;
            };
            // the chunk's residual (fwd) or other-contribution + mask (dgrad) rows are issued at the
            // end of the previous chunk, so their latency overlaps the TMEM load and transpose
            uint4 o1[4];
            uint32_t o2 = 0xFFFFFFFFu;
            auto load_ops = [&](int c, uint4* x1, uint32_t& x2) {
                bool pv;
                const int64_t ro = row_of(c, pv);
#pragma unroll
                for (int i = 0; i < 4; ++i) x1[i] = make_uint4(0u, 0u, 0u, 0u);
                x2 = 0xFFFFFFFFu;
                if (!pv || !active) return;
                const uint4* p1 = reinterpret_cast<const uint4*>((MODE == 0 ? a.res : a.addsrc) + so + ro + ch0);
                if (MODE == 0 ? a.res != nullptr : a.addsrc != nullptr) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) x1[i] = MODE == 0 ? __ldg(p1 + i) : p1[i];
                }
                if (MODE == 1 && a.mbits) x2 = __ldg(a.mbits + ((so + ro + ch0) >> 5));
            };
            load_ops(c_first, o1, o2);  // independent of the accumulator: in flight while the MMAs finish
#ifdef C3_PROF
            const long long q3 = clock64();
#endif
            epi_wait(&tfull[buf], (tl / NBUF) & 1);
#ifdef C3_PROF
            p_tfull += clock64() - q3;
#endif
            tc_fence_after();
            for (int c = c_first; c < 8; c += c_step) {  // 32 pixels per chunk
                float v[32];
                __syncwarp();
                if (nkb > 0) {
                    tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 256 + c * 32, v);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.0f;
                }
                if (!active) continue;
                // v[j] = channel (ch0 + lane) at pixel 32c + j (+ its bias)  →  tr[j][lane]
#pragma unroll
                for (int j = 0; j < 32; ++j) tr[j * kTransPitch + lane] = v[j] + bias;
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = tr[lane * kTransPitch + j];
                __syncwarp();
                bool pv;
                const int64_t rowoff = row_of(c, pv);
                epi_apply32<MODE>(a, v, pv, rowoff, so, ch0, o1, o2);
                if (c + c_step < 8) load_ops(c + c_step, o1, o2);  // in flight during the next TMEM load
                if (MODE == 1 && a.bpart) bsum += warp_transpose_sum(v, lane);
            }
            if (MODE == 1 && a.bpart) {  // combine the warps of each channel group in a fixed order
                float* red = bred + (tl & 1) * NEPI * 32;
                red[warp * 32 + lane] = bsum;
                asm volatile("bar.sync 1, %0;" ::"r"(NEPI * 32) : "memory");
                if (active && warp < (dup ? 2 : 4)) {
                    float t2 = 0.0f;
                    for (int w = cg; w < NEPI; w += (dup ? 2 : 4)) t2 += red[w * 32 + lane];
                    a.bpart[(int64_t)g.s * a.bpart_stride_s + (int64_t)(g.cls * ptiles + g.ptile) * a.C + ch0 +
                            lane] = t2;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
#ifdef C3_PROF
    if ((blockIdx.x == 0 || blockIdx.x == 77) && lane == 0 && (warp == WMMA || warp == WTMA || warp == 0 || warp == 4))
        printf("c3<%d,%d> cta %d warp %d total %lld wait_empty %lld wait_tempty %lld wait_full %lld wait_tfull %lld\n", MODE,
               (int)HALO, blockIdx.x, warp, clock64() - p_start, p_empty, p_tempty, p_full, p_tfull);
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, NBUF * 256);
    }
}

int conv3_halo_ok(int H, int W) {  // the padded window of a 256-pixel tile fits one window stage
    const int PWp = W + 2;
    const int rows = (256 + 2 * PWp + 2 + PWp - 1) / PWp + 1;
    return H >= 1 && rows * PWp * 128 <= c3::kWin ? 1 : 0;
}

int conv3_dgrad_parts(const Conv2Args& a) {
    if (a.halo) return (a.B * (a.H + 1) * (a.W + 2) + 255) / 256;
    const int P = a.B * (a.H / a.stride) * (a.W / a.stride);
    return a.stride * a.stride * ((P + 255) / 256);
}

template <int MODE, bool HALO>
static void launch_conv3_t(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(conv3_kernel<MODE, HALO>), HALO ? c3::kSmemH : c3::kSmem);
    const int ncls = MODE == 1 ? a.stride * a.stride : 1;
    const int PH = MODE == 0 ? a.OH : a.H / a.stride, PW = MODE == 0 ? a.OW : a.W / a.stride;
    const int P = HALO ? a.B * (PH + 1) * (PW + 2) : a.B * PH * PW;
    const int Mtot = MODE == 0 ? a.CO : a.C;
    const int T = a.S * ncls * ((P + 255) / 256) * ((Mtot + 127) / 128);
    Conv2Args b = a;
    b.dbg = conv_debug();
    conv3_kernel<MODE, HALO><<<std::min(T, kNumSMs), HALO ? c3::kThreadsH : c3::kThreads,
                               HALO ? c3::kSmemH : c3::kSmem, st>>>(wmap, bmap, b);
}

template <int MODE>
static void launch_conv3(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    if (a.halo)
        launch_conv3_t<MODE, true>(wmap, bmap, a, st);
    else
        launch_conv3_t<MODE, false>(wmap, bmap, a, st);
}

void launch_conv3_fwd(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv3<0>(wmap, bmap, a, st);
}
void launch_conv3_dgrad(const CUtensorMap& wmapT, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv3<1>(wmapT, bmap, a, st);
}

// ============================================================================ wgrad
// parameter columns of the partials: tap·C + ci, or for the stem (C_pad < 64) the padded
// 8-taps × 8-channels blocks of the forward's K layout (tap·8 + ci, rounded up to 64)
__host__ __device__ inline int conv2_wgrad_cols(const ConvWgradArgs& a) {
    return a.C_pad < 64 ? ((a.k * a.k + 7) / 8) * 64 : a.k * a.k * a.C;  // = conv2_wgrad_cols(taps, C, C_pad)
}

namespace w2 {
constexpr int kEpiWarps = 8;
constexpr int kGatherWarps = 4;
constexpr int kThreads = (kEpiWarps + kGatherWarps + 2) * 32;
constexpr int kData = 216 * 1024;      // stages: as many (A 2 blocks + B 4 blocks of kpx·128 B) as fit
constexpr int kSmem = 1024 + kData + 512;
}  // namespace w2

// Persistent: unit u = (((s·nsplit + split)·co_tiles + ct)·ntiles + nt); neighbouring CTAs share
// (s, split) so the dY and X blocks they read are L2 hits. D[co][col] accumulates in TMEM
// (two 256-column buffers: unit i's store overlaps unit i+1's main loop).
// CPS CTAs per SM: 1 (216 KB of stages, two TMEM accumulators) or 2 (100 KB, one accumulator each:
// two MMA issue streams per SM — one issuing thread sustains ≈ 185 cycles per MMA whatever N,
// profiles/r02/mma_bench*.txt)
template <int CPS>
__global__ void __launch_bounds__(w2::kThreads, CPS)
    conv2_wgrad_kernel(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap xmap,
                       const ConvWgradArgs a, const int g_max_stages_arg) {
    using namespace w2;
    constexpr int NB = CPS == 1 ? 2 : 1;                      // TMEM accumulators of 256 columns
    constexpr int DATA = CPS == 1 ? kData : 100 * 1024;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment as an offset into the __shared__ array: the pointer keeps the shared
    // address space, so plain loads/stores through it compile to LDS/STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    // k-step = kpx pixels (64, or 128 for 64-channel stride-1 layers: half the TMA ops per byte);
    // one 64-wide MN block of an operand is kpx K-rows × 128 B
    const int kpx = a.kpx;
    const int blkB = kpx * 128;
    const int kAStage = 2 * blkB;  // dYᵀ: up to 2 co blocks
    const int kBStage = 4 * blkB;  // X windows: up to 256 parameter columns
    const int kStages = min(g_max_stages_arg, DATA / (kAStage + kBStage));
    uint8_t* sB = smem + kStages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Kt = conv2_wgrad_cols(a);
    // column tiles of 256 (the last one may be narrower: 64 … 256), one MMA width per unit
    const int ntiles = (Kt + 255) / 256, co_tiles = (a.CO + 127) / 128;
    const int npix = a.B * a.OH * a.OW;
    const int nblk_all = (npix + kpx - 1) / kpx;
    const int per = (nblk_all + a.nsplit - 1) / a.nsplit;
    const int T = a.S * a.nsplit * co_tiles * ntiles;
    struct U {
        int s, split, ct, nt, blk0, nblk, w;
    };
    auto unit = [&](int t) {
        U u;
        u.nt = t % ntiles;
        t /= ntiles;
        u.ct = t % co_tiles;
        t /= co_tiles;
        u.split = t % a.nsplit;
        u.s = t / a.nsplit;
        u.blk0 = u.split * per;
        u.nblk = max(0, min(nblk_all, u.blk0 + per) - u.blk0);
        u.w = min(256, Kt - u.nt * 256);
        return u;
    };

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
    if (warp == kEpiWarps + kGatherWarps + 1) tmem_alloc(tslot, NB * 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == kEpiWarps + kGatherWarps) {
        // ------------------------------------------------ TMA: dYᵀ blocks (+ X windows, stride 1)
        if (lane == 0) {
            tma_prefetch_desc(&gmap);
            if (a.tma_b) tma_prefetch_desc(&xmap);
            int it = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const U u = unit(t);
                const int nb = u.w / 64;
                const uint32_t bytes = (a.CO >= 128 ? 2 : 1) * blkB + (a.tma_b ? nb * blkB : 0);
                const int co0 = u.ct * 128;
                for (int b = 0; b < u.nblk; ++b, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_role(&empty[st], ph ^ 1);
                    if (a.dbg & 2) {  // feed-rate experiment: no loads
                        mbar_arrive_expect_tx(&full[st], 0);
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[st], bytes);
                    uint8_t* dst = sA + st * kAStage;
                    const int pix0 = (u.blk0 + b) * kpx;
                    tma_load_4d(&gmap, &full[st], dst, 0, pix0, co0 / 64, u.s);  // ≤ 2 co blocks, one op
                    if (a.tma_b) {
                        const int n0 = pix0 / (a.OH * a.OW), y0 = (pix0 - n0 * a.OH * a.OW) / a.OW;
                        const int cbx = min(nb, a.C / 64);  // channel blocks per op (same tap)
                        for (int j = 0; j < nb; j += cbx) {
                            const int col = u.nt * 256 + 64 * j, tap = col / a.C, ci0 = col - tap * a.C;
                            const int kh = tap / a.k, kw = tap - kh * a.k;
                            // stride 2: the map's W / H element stride is 2 (box = whole output rows)
                            tma_load_5d(&xmap, &full[st], sB + st * kBStage + j * blkB, 0, kw - a.pad,
                                        a.stride * y0 + kh - a.pad, u.s * a.B + n0, ci0 / 64);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == kEpiWarps + kGatherWarps + 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            int it = 0, tl = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
                const U u = unit(t);
                const uint32_t idesc = idesc_bf16(128, u.w, 1, 1);
                const int buf = tl % NB;
                mbar_wait_role(&tempty[buf], ((tl / NB) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                for (int b = 0; b < u.nblk; ++b, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_role(&full[st], ph);
                    if (kAlwaysFence || !(a.tma_b)) fence_proxy_async_smem();  // gathered (generic-proxy) operands only
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + st * kAStage);
                    const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // K = 16 pixels per MMA
                        if (q * 16 >= kpx) break;
                        const uint64_t ad = sdesc_sw128(aBase + 2048 * q, blkB, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 2048 * q, blkB, 1024);
                        if (!(a.dbg & 1)) mma_bf16(d, ad, bd, idesc, (b | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else if (warp >= kEpiWarps) {
        // ------------------------------------------------ gather X windows (stride 2 / stem)
        // thread: 16-byte chunk ch of pixel rows r0 + 16·i; index math hoisted per unit / k-step
        if (!a.tma_b) {
            const int gt = threadIdx.x - kEpiWarps * 32;  // 0..127
            const int ch = gt & 7, r0 = gt >> 3;
            const bool stem = a.C_pad < 64;  // 64 columns = 8 taps × 8 (padded) channels
            const int OHW = a.OH * a.OW;
            int it = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const U u = unit(t);
                const __nv_bfloat16* xs = a.X + u.s * a.X_stride_s;
                int ky[4], kx[4], co_[4];
                const int nb = u.w / 64;
                for (int j = 0; j < nb; ++j) {
                    const int cb = u.nt * 4 + j;
                    int tap, c0;
                    if (stem) {
                        tap = cb * 8 + ch;
                        c0 = 0;
                    } else {
                        tap = (cb * 64) / a.C;
                        c0 = cb * 64 - tap * a.C + 8 * ch;
                    }
                    const int kh = tap / a.k;
                    ky[j] = tap < a.k * a.k ? kh - a.pad : -(1 << 20);  // invalid tap: always OOB
                    kx[j] = tap - kh * a.k - a.pad;
                    co_[j] = c0;
                }
                for (int b = 0; b < u.nblk; ++b, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    int iy0[4], ix0[4];
                    int64_t nb0[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int pix = (u.blk0 + b) * 64 + r0 + 16 * i;
                        const int n = pix / OHW, rem = pix - n * OHW;
                        const int oy = rem / a.OW;
                        iy0[i] = pix < npix ? oy * a.stride : -(1 << 20);
                        ix0[i] = (rem - oy * a.OW) * a.stride;
                        nb0[i] = (int64_t)n * a.H;
                    }
                    gather_wait(&empty[st], ph ^ 1);
                    const uint32_t base = smem_u32(sB + st * kBStage) + ((ch ^ (r0 & 7)) << 4) + r0 * 128;
                    for (int j = 0; j < nb; ++j) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int iy = iy0[i] + ky[j], ix = ix0[i] + kx[j];
                            const bool ok = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                            const __nv_bfloat16* g =
                                ok ? xs + ((nb0[i] + iy) * a.W + ix) * a.C_pad + co_[j] : xs;
                            cp_async16(base + j * 8192 + i * 16 * 128, g, ok ? 16u : 0u);
                        }
                    }
                    cp_async_mbar_arrive(&full[st]);
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue: TMEM → fp32 per-sample partials
        const int q = warp & 3, h = warp >> 2;
        int tl = 0;
        for (int t = blockIdx.x; t < T; t += gridDim.x, ++tl) {
            const U u = unit(t);
            const int buf = tl % NB;
            epi_wait(&tfull[buf], (tl / NB) & 1);
            tc_fence_after();
            const int co = u.ct * 128 + 32 * q + lane;
            const int half = u.w / 2;
            float* out = a.part + ((int64_t)(u.s * a.nsplit + u.split) * a.CO + co) * Kt + u.nt * 256 + h * half;
            for (int c = 0; c < half / 32; ++c) {
                float v[32];
                __syncwarp();
                if (u.nblk > 0) {
                    tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 256 + h * half + 32 * c, v);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.0f;
                }
                if (co < a.CO) {
                    float4* o4 = reinterpret_cast<float4*>(out + 32 * c);
#pragma unroll
                    for (int g = 0; g < 8; ++g) o4[g] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + kGatherWarps + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, NB * 256);
    }
}

int conv2_wgrad_cps() {  // BNN_WGRAD_CPS=1|2 forces the CTAs per SM of the conv2 weight gradient, 0 = per layer
    static int v = [] {
        const char* e = getenv("BNN_WGRAD_CPS");
        const int x = e ? atoi(e) : 0;
        return x == 1 || x == 2 ? x : 0;
    }();
    return v;
}

int conv2_wgrad_ntile(int Kt) { return Kt >= 64 ? 256 : 0; }  // column-tile width (the last may be narrower)

void launch_conv2_wgrad(const CUtensorMap& gmap, const CUtensorMap& xmap, const ConvWgradArgs& a,
                        cudaStream_t st) {
    const int Kt = conv2_wgrad_cols(a);
    const int T = a.S * a.nsplit * ((a.CO + 127) / 128) * ((Kt + 255) / 256);
    ConvWgradArgs b = a;
    b.dbg = conv_debug();
    if (a.kpx == 64 && a.cps == 2) {  // two CTAs per SM (64-pixel k-steps: two 48 KB stages each)
        constexpr int smem = 1024 + 100 * 1024 + 512;
        ensure_smem_attr(reinterpret_cast<const void*>(conv2_wgrad_kernel<2>), smem);
        conv2_wgrad_kernel<2><<<std::min(T, 2 * kNumSMs), w2::kThreads, smem, st>>>(gmap, xmap, b, conv_stage_cap());
        return;
    }
    ensure_smem_attr(reinterpret_cast<const void*>(conv2_wgrad_kernel<1>), w2::kSmem);
    conv2_wgrad_kernel<1><<<std::min(T, kNumSMs), w2::kThreads, w2::kSmem, st>>>(gmap, xmap, b, conv_stage_cap());
}

// Phase 2: thread = four consecutive parameter columns of one row. The partials of up to 8
// samples (and the accumulators) are loaded up front — independent loads, so the kernel
// streams at memory speed — then summed over splits in split order and weighted by ε_s (the
// same EPS-v1 draw as the forward's W_s) in sample order ⇒ deterministic.
__global__ void __launch_bounds__(256)
    wgrad_eps_combine_kernel(SampledLayer L, SampleKeys kk, int S, int nsplit, int CO, int Kt,
                             const float* __restrict__ part, float scale, float* __restrict__ acc_mu,
                             float* __restrict__ acc_rho) {
    const int kq = Kt / 4;
    const int64_t nq = (int64_t)CO * kq;
    const int64_t ss = (int64_t)CO * Kt;  // one split of one sample
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const int co = (int)(i / kq), cq = (int)(i - (int64_t)co * kq);
    const float* p = part + (int64_t)co * Kt + 4 * cq;
    float4* am = reinterpret_cast<float4*>(acc_mu + L.off_w + (int64_t)co * Kt + 4 * cq);
    float4* ar = reinterpret_cast<float4*>(acc_rho + L.off_w + (int64_t)co * Kt + 4 * cq);
    const float4 x0 = *am, y0 = *ar;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f), r = m;
    for (int s0 = 0; s0 < S; s0 += 8) {
        float4 d[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            d[j] = s0 + j < S ? __ldcs(reinterpret_cast<const float4*>(p + (int64_t)(s0 + j) * nsplit * ss))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int sp = 1; sp < nsplit; ++sp) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (s0 + j < S) {
                    const float4 e = __ldcs(reinterpret_cast<const float4*>(p + ((int64_t)(s0 + j) * nsplit + sp) * ss));
                    d[j].x += e.x;
                    d[j].y += e.y;
                    d[j].z += e.z;
                    d[j].w += e.w;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // the 8 Philox chains are independent (ILP); d = 0 past S
            const float4 e = eps4(kk.key, kk.step, kk.s0 + s0 + j, L.t_w, (uint32_t)co, (uint32_t)cq);
            m.x += d[j].x;
            m.y += d[j].y;
            m.z += d[j].z;
            m.w += d[j].w;
            r.x = fmaf(d[j].x, e.x, r.x);
            r.y = fmaf(d[j].y, e.y, r.y);
            r.z = fmaf(d[j].z, e.z, r.z);
            r.w = fmaf(d[j].w, e.w, r.w);
        }
    }
    *am = make_float4(fmaf(scale, m.x, x0.x), fmaf(scale, m.y, x0.y), fmaf(scale, m.z, x0.z), fmaf(scale, m.w, x0.w));
    *ar = make_float4(fmaf(scale, r.x, y0.x), fmaf(scale, r.y, y0.y), fmaf(scale, r.z, y0.z), fmaf(scale, r.w, y0.w));
}

// Small layers (few column quads, many pixel splits): block = 32 column quads × 8 sample lanes;
// a thread sums its (quad, sample) over the splits (four independent chains, fixed order),
// weights by ε_s, and the 8 sample lanes are combined in a fixed order ⇒ deterministic.
__global__ void __launch_bounds__(256)
    wgrad_eps_combine_lanes_kernel(SampledLayer L, SampleKeys kk, int S, int nsplit, int CO, int Kt,
                                   const float* __restrict__ part, float scale, float* __restrict__ acc_mu,
                                   float* __restrict__ acc_rho) {
    __shared__ float4 red[2][8][32];
    const int kq = Kt / 4;
    const int64_t nq = (int64_t)CO * kq;
    const int64_t ss = (int64_t)CO * Kt;
    const int tx = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + tx;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f), r = m;
    int co = 0, cq = 0;
    if (i < nq) {
        co = (int)(i / kq);
        cq = (int)(i - (int64_t)co * kq);
        const float* p = part + (int64_t)co * Kt + 4 * cq;
        for (int s = sl; s < S; s += 8) {
            float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
            const float* ps = p + (int64_t)s * nsplit * ss;
            int sp = 0;
            for (; sp + 2 <= nsplit; sp += 2) {
                const float4 e0 = __ldcs(reinterpret_cast<const float4*>(ps + sp * ss));
                const float4 e1 = __ldcs(reinterpret_cast<const float4*>(ps + (sp + 1) * ss));
                q0.x += e0.x; q0.y += e0.y; q0.z += e0.z; q0.w += e0.w;
                q1.x += e1.x; q1.y += e1.y; q1.z += e1.z; q1.w += e1.w;
            }
            if (sp < nsplit) {
                const float4 e0 = __ldcs(reinterpret_cast<const float4*>(ps + sp * ss));
                q0.x += e0.x; q0.y += e0.y; q0.z += e0.z; q0.w += e0.w;
            }
            const float4 d = make_float4(q0.x + q1.x, q0.y + q1.y, q0.z + q1.z, q0.w + q1.w);
            const float4 e = eps4(kk.key, kk.step, kk.s0 + s, L.t_w, (uint32_t)co, (uint32_t)cq);
            m.x += d.x; m.y += d.y; m.z += d.z; m.w += d.w;
            r.x = fmaf(d.x, e.x, r.x); r.y = fmaf(d.y, e.y, r.y);
            r.z = fmaf(d.z, e.z, r.z); r.w = fmaf(d.w, e.w, r.w);
        }
    }
    red[0][sl][tx] = m;
    red[1][sl][tx] = r;
    __syncthreads();
    if (sl == 0 && i < nq) {
        for (int j = 1; j < 8; ++j) {
            const float4 a = red[0][j][tx], b = red[1][j][tx];
            m.x += a.x; m.y += a.y; m.z += a.z; m.w += a.w;
            r.x += b.x; r.y += b.y; r.z += b.z; r.w += b.w;
        }
        float4* am = reinterpret_cast<float4*>(acc_mu + L.off_w + (int64_t)co * Kt + 4 * cq);
        float4* ar = reinterpret_cast<float4*>(acc_rho + L.off_w + (int64_t)co * Kt + 4 * cq);
        const float4 x0 = *am, y0 = *ar;
        *am = make_float4(fmaf(scale, m.x, x0.x), fmaf(scale, m.y, x0.y), fmaf(scale, m.z, x0.z), fmaf(scale, m.w, x0.w));
        *ar = make_float4(fmaf(scale, r.x, y0.x), fmaf(scale, r.y, y0.y), fmaf(scale, r.z, y0.z), fmaf(scale, r.w, y0.w));
    }
}

// The stem: partial columns are the padded tap·8 + ci, parameter columns tap·C + ci. Block =
// 32 parameters × 8 sample lanes; each thread sums its (parameter, sample) over the splits
// (four independent chains, fixed order), the sample lanes are combined in a fixed order.
__global__ void __launch_bounds__(256)
    wgrad_eps_combine_stem_kernel(SampledLayer L, SampleKeys kk, int S, int nsplit, int CO, int taps, int C,
                                  int Ktp, const float* __restrict__ part, float scale,
                                  float* __restrict__ acc_mu, float* __restrict__ acc_rho) {
    __shared__ float red[2][8][33];
    const int Kt = taps * C;
    const int64_t n = (int64_t)CO * Kt;
    const int tx = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + tx;
    float m = 0.0f, r = 0.0f;
    int co = 0, col = 0;
    if (i < n) {
        co = (int)(i / Kt);
        col = (int)(i - (int64_t)co * Kt);
        const int tap = col / C, pc = tap * 8 + (col - tap * C);
        for (int s = sl; s < S; s += 8) {
            const float* p = part + ((int64_t)s * nsplit * CO + co) * Ktp + pc;
            const int64_t st = (int64_t)CO * Ktp;
            float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
            int sp = 0;
            for (; sp + 4 <= nsplit; sp += 4) {
                q0 += __ldcs(p + sp * st);
                q1 += __ldcs(p + (sp + 1) * st);
                q2 += __ldcs(p + (sp + 2) * st);
                q3 += __ldcs(p + (sp + 3) * st);
            }
            for (; sp < nsplit; ++sp) q0 += __ldcs(p + sp * st);
            const float d = (q0 + q1) + (q2 + q3);
            m += d;
            r = fmaf(d, eps1(kk.key, kk.step, kk.s0 + s, L.t_w, (uint32_t)co, (uint32_t)col), r);
        }
    }
    red[0][sl][tx] = m;
    red[1][sl][tx] = r;
    __syncthreads();
    if (sl == 0 && i < n) {
        for (int j = 1; j < 8; ++j) {
            m += red[0][j][tx];
            r += red[1][j][tx];
        }
        acc_mu[L.off_w + i] = fmaf(scale, m, acc_mu[L.off_w + i]);
        acc_rho[L.off_w + i] = fmaf(scale, r, acc_rho[L.off_w + i]);
    }
}

void launch_wgrad_eps_combine_stem(const SampledLayer& L, const SampleKeys& kk, int S, int nsplit, int CO, int taps,
                                   int C, int Ktp, const float* part, float scale, float* acc_mu, float* acc_rho,
                                   cudaStream_t st) {
    const int64_t n = (int64_t)CO * taps * C;
    wgrad_eps_combine_stem_kernel<<<(int)((n + 31) / 32), 256, 0, st>>>(L, kk, S, nsplit, CO, taps, C, Ktp, part,
                                                                        scale, acc_mu, acc_rho);
}

// nsplit for `base` units per split: fewest waves per split (persistent grid of 148), and among
// choices within 3 % of the best, the fewest splits (each split adds partial traffic)
int conv2_wgrad_nsplit(int base, int blocks, int cps) {  // slots = cps CTAs per SM
    const int slots = std::max(1, cps) * kNumSMs;
    double best = 1e30;
    const int hi = std::max(1, std::min(blocks, 512));
    for (int ns = 1; ns <= hi; ++ns) {
        const int waves = (base * ns + slots - 1) / slots;
        best = std::min(best, (double)waves / ns);
    }
    for (int ns = 1; ns <= hi; ++ns) {
        const int waves = (base * ns + slots - 1) / slots;
        if ((double)waves / ns <= best * 1.03) return ns;
    }
    return hi;
}

void launch_wgrad_eps_combine(const SampledLayer& L, const SampleKeys& kk, int S, int nsplit, int CO, int Kt,
                              const float* part, float scale, float* acc_mu, float* acc_rho, cudaStream_t st) {
    const int64_t nq = (int64_t)CO * Kt / 4;
    if (nq < (int64_t)kNumSMs * 256 && nsplit > 1) {  // few quads: spread the samples over lanes too
        wgrad_eps_combine_lanes_kernel<<<(int)((nq + 31) / 32), 256, 0, st>>>(L, kk, S, nsplit, CO, Kt, part, scale,
                                                                              acc_mu, acc_rho);
        return;
    }
    wgrad_eps_combine_kernel<<<(int)((nq + 255) / 256), 256, 0, st>>>(L, kk, S, nsplit, CO, Kt, part, scale, acc_mu,
                                                                     acc_rho);
}

}  // namespace bnn
