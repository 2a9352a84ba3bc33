// kernels_conv64.cu — W-stationary, row-packed tcgen05 convolution for the stride-1 3×3
// 64 → 64-channel layers (the ResNet's stage 1), forward (K3) and data gradient (K4):
//
//   fwd   Y[p][co]  = Σ_{kh,kw,ci} X[p ⊕ (kh−1, kw−1)][ci] · W_s[co][kh,kw,ci]
//   dgrad dX[p][ci] = Σ_{kh,kw,co} dY[p ⊖ (kh−1, kw−1)][co] · W_s[co][kh,kw,ci]
//
// Why a separate kernel: with 64 output channels the conv3 tile (M = 128
// channels × N = 256 pixels) duplicates its 64 weight rows, so half of every MMA is wasted, the
// 16 KB weight k-blocks are re-read from L2 for every pixel tile (≈ 646 MB of the 877 MB L2→SM
// traffic of a stage-1 dgrad launch, profiles/r02/ncu), and its channel-major accumulator needs
// a shared-memory transpose per 32 × 32 block before the NHWC epilogue.
//
//  * W-stationary: the sample's 9 tap blocks (64 × 64 bf16 each, 72 KB) are loaded ONCE per CTA
//    into resident shared memory; a CTA walks a contiguous range of (sample, pixel tile), so it
//    reloads them at most once (when its range crosses a sample boundary). Only the halo
//    windows stream (≤ 30 KB of whole padded rows per 128-pixel tile, a ring of 4).
//  * Row packing: pixels on M (128 consecutive positions of the padded pixel stream, one halo
//    window), and the three taps of one kernel row (dh, dw = −1, 0, +1) side by side on
//    N = 192 (3 × 64 output channels). One MMA group per kernel row, run against the window at
//    the dw = −1 offset, puts tap (dh, dw)'s contribution to pixel n − (dw + 1) in TMEM lane n,
//    columns 64(dw + 1) + co: 3 groups × 4 K-steps per tile, all 192 columns useful.
//  * Epilogue (thread = pixel = TMEM lane): out[n] = D[n][0:64] + D[n+1][64:128] + D[n+2][128:192]
//    — two warp shuffles per value; the 2 lanes at each warp boundary take their neighbours'
//    values from a 96-float shared exchange (one named barrier per tile and channel half); a
//    tile outputs 126 of its 128 rows. Then the NHWC row in place: + bias, + residual, ReLU,
//    ReLU bitmask (fwd) / + other contribution, input ReLU mask, bias-gradient partials (dgrad),
//    32 channels = 64 contiguous bytes per thread (the dgrad in passes of 16 channels). Two groups
//    of epilogue warps take alternate tiles.
//  * The weight gradient (below): MN-major views of two halo windows, ε fused in the epilogue and
//    the samples of a thread-block cluster summed over DSMEM.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_conv.cuh"
#include "tc_ptx.cuh"

namespace bnn {

using namespace ptx;

namespace c64 {
// epilogue warps: two groups of 8 (4 lane quarters × 2 channel halves) taking even / odd tiles, so
// each group has two MMA tile-times per epilogue (C64_PROF: a group's epilogue of a tile takes
// ≈ 4.7 K cycles, the MMAs ≈ 2.2 K)
constexpr int kGroups = 2;
constexpr int kThreads = (8 * kGroups + 2) * 32;  // + the TMA warp + the MMA warp
constexpr int kBlk = 64 * 128;                  // one tap block: 64 rows × 64 bf16 (SWIZZLE_128B)
constexpr int kWres = 9 * kBlk;                 // 3 kernel rows × 3 taps (72 KB)
constexpr int kNWin = 4;                        // halo window ring
constexpr int kWin = 240 * 128;                 // one window (7 padded rows × 34 px at 32 × 32)
constexpr int kTileM = 128;                     // MMA rows (pixels of the padded stream)
constexpr int kTileP = 126;                     // output pixels per tile (rows 126, 127: neighbours only)
constexpr int kN = 192;                         // 3 taps × 64 channels
constexpr int kCh = 32;                         // channels per epilogue warp
constexpr int kXb = 2 * 2 * 2 * 4 * 3 * kCh * 4;  // [group][tile parity][channel half][lane quarter][3 × 32]
constexpr int kBred = 2 * 2 * 2 * 4 * kCh * 4;   // [group][tile parity][channel half][lane quarter][32]
constexpr int kBars = 256;
constexpr int kSmem = 1024 + kWres + kNWin * kWin + kXb + kBred + kBars;
static_assert(kSmem <= 227 * 1024, "conv64 shared memory");
}  // namespace c64

__host__ __device__ __forceinline__ int c64_floor_div(int a, int b) {  // b > 0
    const int q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

// v of lane + d, or `other` where lane + d is past the warp (shfl's in-range predicate selects)
__device__ __forceinline__ float shfl_down_or(float v, int d, float other) {
    float r;
    asm(
        "{\n\t.reg .pred p;\n\t.reg .f32 t;\n\t"
        "shfl.sync.down.b32 t|p, %1, %2, 0x1f, 0xffffffff;\n\t"
        "selp.f32 %0, t, %3, p;\n\t}"
        : "=f"(r)
        : "f"(v), "r"(d), "f"(other));
    return r;
}

// 32-byte global load / store (LDG.256 / STG.256: one full sector per lane)
template <bool NC>
__device__ __forceinline__ void ld256(const void* p, uint32_t* r) {
    if (NC)
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "l"(p));
    else
        asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st256(void* p, const uint32_t* r) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 16 values whose lanes l and l ^ 16 are equal: lane j (j < 16) ends with Σ over a 16-lane half
// of v[j] (fixed butterfly order)
__device__ __forceinline__ float c64_transpose_sum16(float* v, int lane) {
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = hi ? v[i] : v[i + off];
            const float keep = hi ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// lane j ends with Σ over the warp's 32 lanes of v[j] (fixed butterfly order)
__device__ __forceinline__ float c64_transpose_sum(float* v, int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = hi ? v[i] : v[i + off];
            const float keep = hi ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// C64_PROF (experiment builds, BNN_NVCC_FLAGS=-DC64_PROF): per-role phase cycle sums printed by
// CTA 0 at exit — where a tile's time goes
#ifdef C64_PROF
#define C64_T(x) const long long x = clock64()
#else
#define C64_T(x)
#endif
#ifdef C64_LANE0_MMA
#define C64_MMA mma_bf16
#define C64_COMMIT mma_commit
#else
#define C64_MMA mma_bf16_warp
#define C64_COMMIT mma_commit_warp
#endif

template <int MODE>
__global__ void __launch_bounds__(c64::kThreads, 1)
    conv64_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ Conv64RowMaps rows,
                  const Conv2Args a) {
    using namespace c64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sW = smem;
    uint8_t* sWin = sW + kWres;
    float* xb = reinterpret_cast<float*>(sWin + kNWin * kWin);
    float* bred = xb + kXb / 4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(bred + kBred / 4);
    uint64_t* wres_full = bars;
    uint64_t* wres_empty = bars + 1;
    uint64_t* wfull = bars + 2;            // [kNWin] halo windows
    uint64_t* wempty = bars + 2 + kNWin;   // [kNWin]
    uint64_t* tfull = bars + 2 + 2 * kNWin;  // [2] TMEM accumulators
    uint64_t* tempty = tfull + 2;          // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

    constexpr int NG = kGroups;
    constexpr int WTMA = 8 * NG, WMMA = WTMA + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int PH = a.H, PW = a.W;  // stride 1, pad 1: the output grid is the input grid
    const int PWp = PW + 2, PHp = PH + 1;
    const int ptiles = (a.B * PHp * PWp + kTileP - 1) / kTileP;
    const int64_t T = (int64_t)a.S * ptiles;
    const int t0 = (int)(T * blockIdx.x / gridDim.x), t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);

    if (threadIdx.x == 0) {
        mbar_init(wres_full, 1);
        mbar_init(wres_empty, 1);
        for (int i = 0; i < kNWin; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
        }
        mbar_fence_init();
    }
    if (warp == WMMA) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
#ifdef C64_PROF
    long long p_tma_wait = 0, p_mma_tempty = 0, p_mma_wfull = 0, p_e_wait = 0, p_e_tmem = 0, p_e_bar = 0, p_e_post = 0;
    int p_tiles = 0;
    const long long p_start = clock64();
#endif

    if (warp == WTMA) {
        // ------------------------------------------------ TMA producer: resident W, windows
        if (lane == 0) {
            tma_prefetch_desc(&wmap);
            const CUtensorMap* bm = MODE == 0 ? rows.x : rows.y;  // the window operand: X (fwd) / dY (dgrad)
            int cur_s = -1, seg = 0, tl = 0;
            for (int t = t0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                if (s != cur_s) {  // this sample's 9 tap blocks (after the previous sample's MMAs)
                    if (seg > 0) mbar_wait_role(wres_empty, (seg - 1) & 1);
                    mbar_arrive_expect_tx(wres_full, 9 * kBlk);
                    for (int tap = 0; tap < 9; ++tap) {
                        const int kh = tap / 3, kw = tap - 3 * kh;
                        const int dh = MODE == 0 ? kh - 1 : 1 - kh, dw = MODE == 0 ? kw - 1 : 1 - kw;
                        uint8_t* dst = sW + (3 * (dh + 1) + dw + 1) * kBlk;  // kernel row dh: dw = −1, 0, +1
                        if (MODE == 0)
                            tma_load_3d(&wmap, wres_full, dst, tap * 64, 0, s);  // [co][ci]: K-major B
                        else
                            tma_load_5d(&wmap, wres_full, dst, 0, tap, 0, 0, s);  // [co][ci]: MN-major B
                    }
                    cur_s = s;
                    ++seg;
                }
                const int ws = tl % kNWin;
                C64_T(pa0);
                mbar_wait_role(&wempty[ws], ((tl / kNWin) & 1) ^ 1);
                C64_T(pa1);
#ifdef C64_PROF
                p_tma_wait += pa1 - pa0;
#endif
                const int p0 = pt * kTileP;
                const int rs = c64_floor_div(p0 - PWp - 1, PWp), re = c64_floor_div(p0 + kTileM + PWp, PWp);
                uint8_t* win = sWin + ws * kWin;
                mbar_arrive_expect_tx(&wfull[ws], (uint32_t)((re - rs + 1) * PWp * 128));
                for (int r = rs; r <= re;) {  // one op per run of padded rows inside one image
                    const int b = c64_floor_div(r, PHp), y = r - b * PHp;  // y == PH: separator (OOB: zeros)
#ifdef C64_ROWS1  // A/B: one op per row
                    const int run = 1;
#else
                    const int run = min(min(re, b * PHp + PH) - r + 1, min(8, PH));
#endif
                    tma_load_5d(&bm[run - 1], &wfull[ws], win + (r - rs) * PWp * 128, 0, -1, y, b, s);
                    r += run;
                }
            }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        // ------------------------------------------------ MMA issuer: 3 kernel rows × 4 K-steps per tile
#ifdef C64_LANE0_MMA  // A/B switch: lane 0 alone runs the loop
        if (lane == 0)
#endif
        {  // the whole warp runs the loop (warp-uniform descriptor arithmetic), one lane issues
            const uint32_t idesc = idesc_bf16(kTileM, kN, 0, MODE == 1 ? 1 : 0);
            int cur_s = -1, seg = 0, tl = 0;
            for (int t = t0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                if (s != cur_s) {
                    mbar_wait_role(wres_full, seg & 1);
                    cur_s = s;
                    ++seg;
                }
                const int buf = tl & 1, ws = tl % kNWin;
                C64_T(pm0);
                mbar_wait_role(&tempty[buf], ((tl >> 1) & 1) ^ 1);
                C64_T(pm1);
                mbar_wait_role(&wfull[ws], (tl / kNWin) & 1);
                C64_T(pm2);
#ifdef C64_PROF
                p_mma_tempty += pm1 - pm0;
                p_mma_wfull += pm2 - pm1;
#endif
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                const int p0 = pt * kTileP;
                const int wrow0 = p0 - c64_floor_div(p0 - PWp - 1, PWp) * PWp;  // window row of pixel p0
                const uint32_t winb = smem_u32(sWin + ws * kWin);
                // descriptors of the (g, q) = (0, 0) operands; the others add their byte offset ÷ 16 to the
                // start-address field (the smem addresses stay below 256 KB: no carry out of the field)
                const uint64_t ad0 = sdesc_sw128(winb + (uint32_t)(wrow0 - PWp - 1) * 128u, 16, 1024);
                const uint64_t bd0 = MODE == 0 ? sdesc_sw128(smem_u32(sW), 16, 1024) : sdesc_sw128(smem_u32(sW), kBlk, 1024);
#pragma unroll
                for (int g = 0; g < 3; ++g) {  // kernel row dh = g − 1, window at its dw = −1 tap
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = ad0 + (uint64_t)(g * PWp * 8 + 2 * q);
                        const uint64_t bd = bd0 + (uint64_t)((3 * g * kBlk) / 16 + (MODE == 0 ? 2 * q : 128 * q));
                        C64_MMA(d, ad, bd, idesc, (g | q) != 0 ? 1u : 0u);
                    }
                }
                C64_COMMIT(&wempty[ws]);
                C64_COMMIT(&tfull[buf]);
                if (t + 1 < t1 && (t + 1) / ptiles != s) C64_COMMIT(wres_empty);  // W free for the next sample
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue: group g = warp / 8 takes the tiles
        // of TMEM buffer g (every other tile of the CTA: each group has two MMA tile-times per
        // epilogue); warp (q, h) = TMEM lane quarter q (pixels 32q … 32q+31), channels 32h … 32h+31
        const int g = warp >> 3, q = warp & 3, h = (warp >> 2) & 1;
        const int bar_id = 1 + 2 * g + h;
        const int ch0 = kCh * h;
        const int m = 32 * q + lane;  // tile row = pixel offset
        // x / PWp and x / PHp as a multiply-shift (x < 2^24: exact with a 40-bit reciprocal)
        const uint64_t mW = ((1ull << 40) + PWp - 1) / PWp, mH = ((1ull << 40) + PHp - 1) / PHp;
        int prev_s = 0, prev_pt = 0;
        int tl = g;
        for (int t = t0 + g; t < t1; t += NG, tl += NG) {
            const int s = t / ptiles, pt = t - s * ptiles;
            const int buf = tl & 1, par = (tl / NG) & 1;
            const int64_t so = (int64_t)s * a.out_stride_s;
            const int pix = pt * kTileP + m;
            const int r = (int)(((uint64_t)pix * mW) >> 40), cx = pix - r * PWp;
            const int b = (int)(((uint64_t)r * mH) >> 40), y = r - b * PHp;
            const bool pv = m < kTileP && b < a.B && y < PH && cx >= 1 && cx <= PW;
            const int64_t ro = pv ? (((int64_t)b * PH + y) * PW + cx - 1) * 64 + ch0 : 0;
            uint32_t xw[16];  // 32 bf16 of the residual / other contribution: two 32-byte loads
#pragma unroll
            for (int i = 0; i < 16; ++i) xw[i] = 0u;
            uint32_t mw = 0xFFFFFFFFu;
            const __nv_bfloat16* opnd = MODE == 0 ? a.res : a.addsrc;
            if (pv && opnd) {  // the row's residual / other contribution, in flight during the wait
                ld256<MODE == 0>(opnd + so + ro, xw);  // dgrad: the contribution may be the output buffer
                ld256<MODE == 0>(opnd + so + ro + 16, xw + 8);
            }
            if (MODE == 1 && pv && a.mbits) mw = __ldg(a.mbits + ((so + ro) >> 5));
            C64_T(pe0);
            epi_wait(&tfull[buf], (tl >> 1) & 1);  // the other group works meanwhile
            C64_T(pe1);
            tc_fence_after();
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 256 + ch0;
            // Passes of CH channels (dgrad: 16, the register budget of 18 warps with the bias-gradient
            // butterfly; fwd: 32). xq: [0] row 0's dw = +1 block, [1] row 0's dw = 0 block, [2] row 1's
            // dw = +1 block — what the previous quarter's rows 30, 31 need from this one.
            constexpr int CH = MODE == 1 ? 16 : 32;
            float* xq = xb + (((g * 2 + par) * 2 + h) * 4 + q) * 3 * kCh;
#pragma unroll
            for (int c0 = 0; c0 < kCh; c0 += CH) {
                float z[CH], v[16];
#pragma unroll
                for (int c = c0; c < c0 + CH; c += 16) {
                    tmem_ld16(ta + c, z + (c - c0));  // block dw = −1 (this pixel)
                    tmem_ld16(ta + 64 + c, v);         // dw = 0 (pixel − 1)
                    if (q > 0 && lane == 0) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(xq + kCh + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j) z[c - c0 + j] += shfl_down_or(v[j], 1, 0.0f);
                    tmem_ld16(ta + 128 + c, v);        // dw = +1 (pixel − 2)
                    if (c + 16 == kCh) {  // the tile's last accumulator read
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    if (q > 0 && lane < 2) {
                        float* d = xq + (lane == 0 ? 0 : 2 * kCh) + c;
#pragma unroll
                        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j) z[c - c0 + j] += shfl_down_or(v[j], 2, 0.0f);
                }
                C64_T(pe2);
                named_bar(bar_id, 4 * 32);  // the exchange of this pass is written
                C64_T(pe3);
#ifdef C64_PROF
                if (c0 == 0) {
                    p_e_tmem += pe2 - pe1;
                    p_e_bar += pe3 - pe2;
                }
#endif
                if (q < 3 && lane >= 30) {  // rows 30, 31: the next quarter's rows 0, 1 (same summation order)
                    const float* xn = xb + (((g * 2 + par) * 2 + h) * 4 + q + 1) * 3 * kCh + c0;
                    if (lane == 31) {
#pragma unroll
                        for (int j = 0; j < CH; j += 4) {
                            const float4 fb = *reinterpret_cast<const float4*>(xn + kCh + j);
                            const float4 fc = *reinterpret_cast<const float4*>(xn + 2 * kCh + j);
                            z[j] = (z[j] + fb.x) + fc.x;
                            z[j + 1] = (z[j + 1] + fb.y) + fc.y;
                            z[j + 2] = (z[j + 2] + fb.z) + fc.z;
                            z[j + 3] = (z[j + 3] + fb.w) + fc.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < CH; j += 4) {
                            const float4 fc = *reinterpret_cast<const float4*>(xn + j);
                            z[j] += fc.x;
                            z[j + 1] += fc.y;
                            z[j + 2] += fc.z;
                            z[j + 3] += fc.w;
                        }
                    }
                }
                if (MODE == 1 && a.bpart && c0 == 0 && t > t0 + g && q == 0) {  // this group's previous tile
                    const float* rb = bred + ((g * 2 + (par ^ 1)) * 2 + h) * 4 * kCh;
                    a.bpart[(int64_t)prev_s * a.bpart_stride_s + (int64_t)prev_pt * a.C + ch0 + lane] =
                        ((rb[lane] + rb[kCh + lane]) + rb[2 * kCh + lane]) + rb[3 * kCh + lane];
                }
                if (pv) {
                    if (MODE == 0) {
                        const float4* bs = reinterpret_cast<const float4*>(a.bias + (int64_t)s * a.CO + ch0 + c0);
#pragma unroll
                        for (int k = 0; k < CH / 4; ++k) {
                            const float4 b4 = __ldg(bs + k);
                            z[4 * k] += b4.x;
                            z[4 * k + 1] += b4.y;
                            z[4 * k + 2] += b4.z;
                            z[4 * k + 3] += b4.w;
                        }
                    }
                    if (opnd) {
#pragma unroll
                        for (int e = 0; e < CH / 2; ++e) {
                            const uint32_t wv = xw[c0 / 2 + e];
                            z[2 * e] += __uint_as_float(wv << 16);
                            z[2 * e + 1] += __uint_as_float(wv & 0xFFFF0000u);
                        }
                    }
                    if (MODE == 0) {
                        if (a.relu) {
#pragma unroll
                            for (int j = 0; j < CH; ++j) z[j] = fmaxf(z[j], 0.0f);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (!((mw >> (c0 + j)) & 1u)) z[j] = 0.0f;
                    }
                    uint32_t pk[CH / 2];
#pragma unroll
                    for (int k = 0; k < CH / 2; ++k) pk[k] = pack_bf16x2(z[2 * k], z[2 * k + 1]);
#pragma unroll
                    for (int k = 0; k < CH / 16; ++k) st256(a.out + so + ro + c0 + 16 * k, pk + 8 * k);  // full sectors
                    if (MODE == 0 && a.mbits_out) {
                        // bit j = (stored bf16 of channel ch0 + j > 0); after the ReLU no stored value is
                        // negative, so > 0 ⟺ magnitude bits ≠ 0: (x & 0x7FFF) + 0x7FFF carries into bit 15
                        uint32_t bits = 0;
#pragma unroll
                        for (int k = 0; k < CH / 2; ++k) {
                            const uint32_t cb = ((pk[k] & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x80008000u;
                            bits |= (((cb >> 15) & 1u) | (cb >> 30)) << (2 * k);  // bit 0: low half, bit 1: high half
                        }
                        a.mbits_out[(so + ro) >> 5] = bits;  // CH = 32: the whole word
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < CH; ++j) z[j] = 0.0f;
                }
                if (MODE == 1 && a.bpart) {  // Σ over the quarter's 32 pixels per channel (fixed order)
                    float* rb = bred + (((g * 2 + par) * 2 + h) * 4 + q) * kCh + c0;
                    if (CH == 32) {
                        const float bsum = c64_transpose_sum(z, lane);  // lane j: channel j of the pass
                        rb[lane] = bsum;
                    } else {
#pragma unroll
                        for (int j = 0; j < CH; ++j) z[j] += __shfl_xor_sync(0xffffffffu, z[j], 16);
                        const float bsum = c64_transpose_sum16(z, lane);  // lanes l, l + 16: channel l & 15
                        if (lane < 16) rb[lane] = bsum;
                    }
                }
            }
            prev_s = s;
            prev_pt = pt;
#ifdef C64_PROF
            C64_T(pe4);
            p_e_wait += pe1 - pe0;
            p_e_post += pe4 - pe1;
            ++p_tiles;
#endif
        }
        if (MODE == 1 && a.bpart && t1 > t0 + g) {  // flush the group's last tile's partials
            named_bar(bar_id, 4 * 32);
            if (q == 0) {
                const float* rb = bred + ((g * 2 + (((tl - NG) / NG) & 1)) * 2 + h) * 4 * kCh;
                a.bpart[(int64_t)prev_s * a.bpart_stride_s + (int64_t)prev_pt * a.C + ch0 + lane] =
                    ((rb[lane] + rb[kCh + lane]) + rb[2 * kCh + lane]) + rb[3 * kCh + lane];
            }
        }
    }
#ifdef C64_PROF
    if ((blockIdx.x == 0 || blockIdx.x == 77) && lane == 0) {
        const long long tot = clock64() - p_start;
        if (warp == WTMA) printf("c64<%d> cta %d TMA: total %lld wait_wempty %lld\n", MODE, blockIdx.x, tot, p_tma_wait);
        else if (warp == WMMA) printf("c64<%d> cta %d MMA: total %lld wait_tempty %lld wait_wfull %lld\n", MODE, blockIdx.x, tot, p_mma_tempty, p_mma_wfull);
        else if ((warp & 3) == 0) printf("c64<%d> cta %d epi warp %d: tiles %d total %lld wait_tfull %lld tmem+shfl %lld bar %lld post %lld\n",
                                      MODE, blockIdx.x, warp, p_tiles, tot, p_e_wait, p_e_tmem, p_e_bar, p_e_post);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ============================================================================ weight gradient
// dW_s[co][kh,kw][ci] = Σ_p dY_s[p][co] · X_s[p ⊕ (kh−1, kw−1)][ci]   (per sample)
// over the padded pixel stream (pad columns and separator rows of dY and X are zero), split into
// contiguous pixel ranges, one (sample, split) per CTA. Both operands come straight out of halo
// windows as MN-major SWIZZLE_128B views (scripts/mn_desc_test.cu, profiles/r02/mn_desc_test.txt):
//   A (M = 128): rows 0–63 = dY[p][co], rows 64–127 = dY[p + 1][co] (second M block one 128-B row
//     later: LBO = 128 B);
//   B (N = 192): X[p + o + j·(W+2)][ci], j = 0, 1, 2 (N blocks one padded row apart).
// With o = −(W+2) + 1 the lower rows give the taps (dh, +1) of the three kernel rows and the upper
// rows, whose dY is one pixel later, the taps (dh, 0); with o = −(W+2) − 1 the lower rows give
// (dh, −1) (upper rows unused). Two N = 192 MMAs per 16 pixels cover all 9 taps (the generic
// conv2 wgrad: three MMAs, N = 256, 256, 64, half of M idle). Output: the fp32 per-sample
// partials part[s][split][co][tap·64 + ci] of the ε combine (kernels_conv2.cu).
namespace c64w {
constexpr int kKpx = 128;                 // pixels per k-block
constexpr int kXw = 240 * 128;            // X window: ≤ 240 padded pixels (7 rows of 34)
constexpr int kYw = 176 * 128;            // dY window: ≤ 176 padded pixels (5 rows of 34)
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int kSmem = 1024 + kStages * (kXw + kYw) + 256;
static_assert(kSmem <= 227 * 1024, "conv64 wgrad shared memory");
}  // namespace c64w

// cluster size of the ε-fused form (a.eps_cluster): by default 2 samples when S is even
// (measured, one B200 with this kernel's 214 KB of shared memory: 15 co-resident clusters of 8 =
// 120 CTAs, 32 of 4 = 128, pairs fill the chip: 156 / 149 / 133 µs per C3 layer), else 1; the
// groups of a split are summed by the split reduce in (split, group) order.
// BNN_WGRAD_EPS_CLUSTER=S (S ≤ 8) sums all samples of a split over DSMEM (no per-group partials).
int conv64_wgrad_eps_cluster(int S) {
    const char* e = getenv("BNN_WGRAD_EPS_CLUSTER");
    if (e) {
        const int g = atoi(e);
        if (g >= 1 && g <= 8 && S % g == 0) return g;
    }
    return S % 2 == 0 ? 2 : 1;
}

// EPS (ε-fused, sample-accumulating): the S samples of one pixel split form a thread-block
// cluster (rank = sample). Each CTA turns its D_s into (D_s, ε_s ⊙ D_s) — ε regenerated, the same
// EPS-v1 draw as the forward's W_s — and leaves them in its shared memory; after a cluster barrier
// CTA j sums rows [j·64/S, (j+1)·64/S) over the S samples in sample order (DSMEM reads) and writes
// scale·Σ to the split partials part[split][μ | ρ][64·576] (wgrad_split_reduce adds the splits in
// order). No per-sample partials, no separate ε combine (north_star (3)); deterministic.
template <bool EPS>
__global__ void __launch_bounds__(c64w::kThreads, 1)
    conv64_wgrad_kernel(const __grid_constant__ Conv64RowMaps maps, const ConvWgradArgs a) {
    using namespace c64w;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * (kXw + kYw));
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
    constexpr int WTMA = kEpiWarps, WMMA = kEpiWarps + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int PH = a.H, PW = a.W, PWp = PW + 2, PHp = PH + 1;
    // EPS: blockIdx = (partial index u = split·groups + group)·Gc + rank, sample = group·Gc + rank;
    // pixel split = u / groups (a.nsplit counts the partials, splits × groups)
    const int Gc = EPS ? a.eps_cluster : 1, groups = a.S / Gc;
    const int s = EPS ? (int)((blockIdx.x / Gc) % groups) * Gc + (int)(blockIdx.x % Gc) : (int)(blockIdx.x / a.nsplit);
    const int u = EPS ? (int)(blockIdx.x / Gc) : (int)(blockIdx.x - s * a.nsplit);
    const int usplit = EPS ? u / groups : u, nsplit_px = EPS ? a.nsplit / groups : a.nsplit;
    const int nkb_all = (a.B * PHp * PWp + kKpx - 1) / kKpx;
    const int kb0 = (int)((int64_t)nkb_all * usplit / nsplit_px), kb1 = (int)((int64_t)nkb_all * (usplit + 1) / nsplit_px);

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_fence_init();
    }
    if (warp == WMMA) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == WTMA) {
        if (lane == 0) {
            // padded rows r0 … r1 to dst: one TMA op per run of rows inside one image (its separator
            // row y = PH and rows of images outside [0, B) are out of range: zeros)
            auto load_rows = [&](const CUtensorMap* m, uint64_t* bar, uint8_t* dst, int r0, int r1) {
                for (int r = r0; r <= r1;) {
                    const int b = c64_floor_div(r, PHp), y = r - b * PHp;
                    const int run = min(min(r1, b * PHp + PH) - r + 1, min(8, PH));  // the maps: 1 … min(8, H) rows
                    tma_load_5d(&m[run - 1], bar, dst + (r - r0) * PWp * 128, 0, -1, y, b, s);
                    r += run;
                }
            };
            for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
                const int st = it % kStages;
                mbar_wait_role(&empty[st], ((it / kStages) & 1) ^ 1);
                const int p0 = kb * kKpx;
                const int xs = c64_floor_div(p0 - PWp - 1, PWp), xe = c64_floor_div(p0 + kKpx + PWp, PWp);
                const int ys = c64_floor_div(p0, PWp), ye = c64_floor_div(p0 + kKpx, PWp);
                uint8_t* xw = smem + st * (kXw + kYw);
                uint8_t* yw = xw + kXw;
                if (a.dbg & 2) {  // timing experiment (BNN_CONV_DEBUG=2): no operand loads
                    mbar_arrive_expect_tx(&full[st], 0);
                    continue;
                }
                mbar_arrive_expect_tx(&full[st], (uint32_t)((xe - xs + 1 + ye - ys + 1) * PWp * 128));
                load_rows(maps.x, &full[st], xw, xs, xe);
                load_rows(maps.y, &full[st], yw, ys, ye);
            }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        // the whole warp runs the loop (warp-uniform descriptor arithmetic), one lane issues
        {
            const uint32_t idesc = idesc_bf16(128, 192, 1, 1);
            for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
                const int st = it % kStages;
                mbar_wait_role(&full[st], (it / kStages) & 1);
                tc_fence_after();
                const int p0 = kb * kKpx;
                const int xs = c64_floor_div(p0 - PWp - 1, PWp), ys = c64_floor_div(p0, PWp);
                const uint32_t xb0 = smem_u32(smem + st * (kXw + kYw)) + (uint32_t)(p0 - xs * PWp) * 128u;
                const uint32_t yb0 = smem_u32(smem + st * (kXw + kYw) + kXw) + (uint32_t)(p0 - ys * PWp) * 128u;
                const uint64_t ad0 = sdesc_sw128(yb0, 128, 1024);
                const uint64_t bA0 = sdesc_sw128(xb0 + (uint32_t)(1 - PWp) * 128u, PWp * 128, 1024);
                const uint64_t bB0 = sdesc_sw128(xb0 - (uint32_t)(1 + PWp) * 128u, PWp * 128, 1024);
#pragma unroll
                for (int q = 0; q < kKpx / 16; ++q) {  // + 2048 B per K-step: + 128 in the address field
                    const uint32_t acc = (it | q) != 0 ? 1u : 0u;
                    if (a.dbg & 1) continue;  // timing experiment (BNN_CONV_DEBUG=1): no MMAs
                    mma_bf16_warp(tmem, ad0 + 128u * q, bA0 + 128u * q, idesc, acc);        // taps (dh, +1) | (dh, 0)
                    mma_bf16_warp(tmem + 256, ad0 + 128u * q, bB0 + 128u * q, idesc, acc);  // taps (dh, −1) | unused
                }
                mma_commit_warp(&empty[st]);
            }
            mma_commit_warp(tfull);
        }
        __syncwarp();
    } else if (!EPS) {
        // epilogue: warp (q, hh) — TMEM lane quarter q (lower rows: co = 32q + lane; upper rows:
        // co = 32(q − 2) + lane), column blocks split between hh = 0, 1
        const int q = warp & 3, hh = warp >> 2;
        const bool upper = q >= 2;
        const int co = 32 * (q & 1) + lane;
        const bool any = kb1 > kb0;
        if (any) {
            epi_wait(tfull, 0);
            tc_fence_after();
        }
        float* outrow = a.part + ((int64_t)(s * a.nsplit + u) * 64 + co) * 576;
        // (accumulator column block, tap) pairs of this warp: lower rows: A blocks j → tap 3j + 2,
        // B blocks j → tap 3j; upper rows: A blocks j → tap 3j + 1
        const int nblk = upper ? 3 : 6;
        for (int i = hh; i < nblk; i += 2) {
            const int j = i % 3;
            const bool tileB = i >= 3;
            const int tap = upper ? 3 * j + 1 : (tileB ? 3 * j : 3 * j + 2);
            float v[32];
#pragma unroll
            for (int c = 0; c < 64; c += 32) {
                __syncwarp();
                if (any) {
                    tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + (tileB ? 256 : 0) + 64 * j + c, v);
                } else {
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = 0.0f;
                }
                float4* o4 = reinterpret_cast<float4*>(outrow + tap * 64 + c);
#pragma unroll
                for (int k = 0; k < 8; ++k) o4[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            }
        }
    }
    if (EPS) {
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        constexpr int kPitch = 196;  // floats per exchange row (conflict-free float4 stores)
        float* xch = reinterpret_cast<float*>(smem);  // [2: D, ε⊙D][64 co][kPitch]: the stage memory, free now
        const bool any = kb1 > kb0;
        const int q = warp & 3, hh = warp >> 2;
        if (warp < kEpiWarps && any) {
            epi_wait(tfull, 0);
            tc_fence_after();
        }
        const int S = Gc;  // the cluster's samples
        const int rank = (int)cluster.block_rank();
        const int rows = (64 + S - 1) / S, r0 = rank * rows, r1 = min(64, r0 + rows);
        const int n = 64 * 576;
        for (int j = 0; j < 3; ++j) {  // kernel row j: taps 3j (tile B lower), 3j+1 (tile A upper), 3j+2 (tile A lower)
            if (warp < kEpiWarps) {
                const bool upper = q >= 2;
                const int co = 32 * (q & 1) + lane;
                const int loc = upper ? 1 : (hh == 0 ? 2 : 0);         // tap 3j + loc
                const uint32_t col0 = (upper ? 0u : (hh == 0 ? 0u : 256u)) + 64 * j;  // accumulator columns
                const int c_lo = upper ? 32 * hh : 0, c_hi = upper ? c_lo + 32 : 64;
                for (int c = c_lo; c < c_hi; c += 32) {
                    float v[32];
                    __syncwarp();
                    if (any) {
                        tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + col0 + c, v);
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k) v[k] = 0.0f;
                    }
                    const uint32_t quad0 = (uint32_t)((3 * j + loc) * 64 + c) / 4;
                    float* xm = xch + co * kPitch + loc * 64 + c;
                    float* xr = xm + 64 * kPitch;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float4 e = eps4(a.kk.key, a.kk.step, a.kk.s0 + s, a.L.t_w, (uint32_t)co, quad0 + k);
                        *reinterpret_cast<float4*>(xm + 4 * k) = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                        *reinterpret_cast<float4*>(xr + 4 * k) =
                            make_float4(v[4 * k] * e.x, v[4 * k + 1] * e.y, v[4 * k + 2] * e.z, v[4 * k + 3] * e.w);
                    }
                }
            }
            cluster.sync();  // every sample's (D, ε ⊙ D) for kernel row j is in its CTA's shared memory
            for (int e = threadIdx.x; e < (r1 - r0) * 48; e += blockDim.x) {  // 4 columns per task
                const int co = r0 + e / 48, cc = 4 * (e - (e / 48) * 48);
                float4 xm[8], xr[8];  // every sample's values in flight at once (S ≤ 8)
#pragma unroll
                for (int rr = 0; rr < 8; ++rr) {
                    if (rr < S) {
                        const float* src = cluster.map_shared_rank(xch, rr);
                        xm[rr] = *reinterpret_cast<const float4*>(src + co * kPitch + cc);
                        xr[rr] = *reinterpret_cast<const float4*>(src + (64 + co) * kPitch + cc);
                    }
                }
                float4 m = make_float4(0.f, 0.f, 0.f, 0.f), r = m;
#pragma unroll
                for (int rr = 0; rr < 8; ++rr) {  // sample order ⇒ deterministic
                    if (rr < S) {
                        m.x += xm[rr].x; m.y += xm[rr].y; m.z += xm[rr].z; m.w += xm[rr].w;
                        r.x += xr[rr].x; r.y += xr[rr].y; r.z += xr[rr].z; r.w += xr[rr].w;
                    }
                }
                const int col = (3 * j + cc / 64) * 64 + (cc & 63);
                const float k = a.scale;
                *reinterpret_cast<float4*>(a.part + (int64_t)u * 2 * n + co * 576 + col) =
                    make_float4(k * m.x, k * m.y, k * m.z, k * m.w);
                *reinterpret_cast<float4*>(a.part + (int64_t)u * 2 * n + n + co * 576 + col) =
                    make_float4(k * r.x, k * r.y, k * r.z, k * r.w);
            }
            cluster.sync();  // the exchange is read before the next row overwrites it
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int conv64_wgrad_ok(int H, int W) {  // both halo windows of a 128-pixel k-block fit their stages
    const int PWp = W + 2;
    const int rx = (c64w::kKpx + 3 * PWp) / PWp + 1, ry = (c64w::kKpx + PWp) / PWp + 1;
    return H >= 1 && rx * PWp * 128 <= c64w::kXw && ry * PWp * 128 <= c64w::kYw ? 1 : 0;
}

int conv64_wgrad_nsplit(int S) { return std::max(1, kNumSMs / std::max(S, 1)); }

void launch_conv64_wgrad(const Conv64RowMaps& maps, const ConvWgradArgs& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(conv64_wgrad_kernel<false>), c64w::kSmem);
    conv64_wgrad_kernel<false><<<a.S * a.nsplit, c64w::kThreads, c64w::kSmem, st>>>(maps, a);
}

static cudaLaunchConfig_t eps_cfg(int Gc, int nparts, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(Gc * nparts), 1, 1);
    cfg.blockDim = dim3(c64w::kThreads, 1, 1);
    cfg.dynamicSmemBytes = c64w::kSmem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)Gc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

int conv64_wgrad_eps_nsplit(int S, int Gc) {  // partials (splits × sample groups) of one co-resident wave, 0 if none
    if (S < 1 || Gc < 1 || S % Gc != 0) return 0;
    ensure_smem_attr(reinterpret_cast<const void*>(conv64_wgrad_kernel<true>), c64w::kSmem);
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = eps_cfg(Gc, 1, nullptr, attr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, conv64_wgrad_kernel<true>, &cfg) != cudaSuccess || n < 1) {
        (void)cudaGetLastError();
        return 0;
    }
    const int groups = S / Gc;
    return std::max(1, n / groups) * groups;  // whole pixel splits: every split has all sample groups
}

int launch_conv64_wgrad_eps(const Conv64RowMaps& maps, const ConvWgradArgs& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(conv64_wgrad_kernel<true>), c64w::kSmem);
    cudaLaunchAttribute attr[1];
    if (a.eps_cluster < 1 || a.S % a.eps_cluster != 0 || a.nsplit % (a.S / a.eps_cluster) != 0) return -1;
    cudaLaunchConfig_t cfg = eps_cfg(a.eps_cluster, a.nsplit, st, attr);
    ConvWgradArgs b = a;
    static const int dbg = [] {  // BNN_CONV_DEBUG (timing experiments): 1 = no MMAs, 2 = no operand loads
        const char* e = getenv("BNN_CONV_DEBUG");
        return e ? atoi(e) : 0;
    }();
    b.dbg = dbg;
    return cudaLaunchKernelEx(&cfg, conv64_wgrad_kernel<true>, maps, b) == cudaSuccess ? 0 : -1;
}

int conv64_ok(int H, int W) {  // the padded window of a 128-row tile fits one window stage
    const int PWp = W + 2;
    const int rows = (c64::kTileM + 3 * PWp) / PWp + 1;
    return H >= 1 && rows * PWp * 128 <= c64::kWin ? 1 : 0;
}

int conv64_parts(const Conv2Args& a) { return (a.B * (a.H + 1) * (a.W + 2) + c64::kTileP - 1) / c64::kTileP; }

template <int MODE>
static void launch_conv64(const CUtensorMap& wmap, const Conv64RowMaps& rows, const Conv2Args& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(conv64_kernel<MODE>), c64::kSmem);
    const int64_t T = (int64_t)a.S * conv64_parts(a);
    conv64_kernel<MODE><<<(int)std::min<int64_t>(T, kNumSMs), c64::kThreads, c64::kSmem, st>>>(wmap, rows, a);
}

void launch_conv64_fwd(const CUtensorMap& wmap, const Conv64RowMaps& rows, const Conv2Args& a, cudaStream_t st) {
    launch_conv64<0>(wmap, rows, a, st);
}
void launch_conv64_dgrad(const CUtensorMap& wmapT, const Conv64RowMaps& rows, const Conv2Args& a, cudaStream_t st) {
    launch_conv64<1>(wmapT, rows, a, st);
}

}  // namespace bnn
