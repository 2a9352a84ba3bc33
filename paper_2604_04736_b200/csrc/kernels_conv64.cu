// kernels_conv64.cu — W-stationary, tap-paired tcgen05 convolution for the stride-1 3×3
// 64 → 64-channel layers (the ResNet's stage 1), forward (K3) and data gradient (K4):
//
//   fwd   Y[p][co]  = Σ_{kh,kw,ci} X[p ⊕ (kh−1, kw−1)][ci] · W_s[co][kh,kw,ci]
//   dgrad dX[p][ci] = Σ_{kh,kw,co} dY[p ⊖ (kh−1, kw−1)][co] · W_s[co][kh,kw,ci]
//
// Why a separate kernel: with 64 output channels the conv3 tile (M = 128
// channels × N = 256 pixels) duplicates its 64 weight rows, so half of every MMA is wasted, and
// the 16 KB weight k-blocks are re-read from L2 for every pixel tile (≈ 646 MB of the 877 MB
// L2→SM traffic of a stage-1 dgrad launch, profiles/r02/ncu).
//
//  * W-stationary: the sample's 9 tap blocks (64 × 64 bf16 each, 72 KB) are loaded ONCE per CTA
//    into resident shared memory; a CTA walks a contiguous range of (sample, pixel tile), so it
//    reloads them at most once (when its range crosses a sample boundary). Only the halo
//    windows stream (one ≈ 47 KB window of whole padded rows per tile, as conv3's HALO tile).
//  * Tap pairing: an M = 128 MMA whose rows 0–63 hold tap a = (dh, −1) and rows 64–127 tap
//    b = (dh, 0) of the same kernel row, run against the window at tap a's offset, puts tap
//    b's contribution to pixel n − 1 in TMEM lane 64 + co, column n (tap b's window offset is
//    tap a's + 1). Three such pairs plus three single taps (dw = +1, rows 64–127 zero) cover
//    the 9 taps in 6 MMA groups instead of 9. A tile computes 256 columns and outputs the 255
//    pixels whose upper contribution it holds: out[n] = L[n] + U[n + 1].
//  * Epilogue: warp q of the TMEM lane quarters (q = 0, 1: lower channels 0–31 / 32–63;
//    q = 2, 3: upper) transposes its 32 channels × 32 columns through shared memory (the upper
//    warps shifted by one column), then each lower/upper warp pair sums the two and finishes
//    the NHWC rows thread = pixel, 16 channels each (+ bias, + residual, ReLU, ReLU bitmask /
//    + other contribution, input ReLU mask, bias-gradient partials), 32-byte stores.
#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_conv.cuh"
#include "tc_ptx.cuh"

namespace bnn {

using namespace ptx;

namespace c64 {
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarps + 2) * 32;  // + the TMA warp + the MMA warp
constexpr int kBlk = 64 * 128;                  // one tap block: 64 rows × 64 bf16 (SWIZZLE_128B)
constexpr int kWres = 12 * kBlk;                // 6 groups of two blocks (3 pairs, 3 singles + zeros)
constexpr int kWin = 374 * 128;                 // one halo window (11 padded rows × 34 px at 32 × 32)
constexpr int kTransPitch = 33;                 // floats per transposed row (conflict-free)
constexpr int kTrans = kEpiWarps * 32 * kTransPitch * 4;
constexpr int kTileN = 255;                     // output pixels per tile (256 MMA columns)
constexpr int kBars = 256;
constexpr int kBred = 2 * kEpiWarps * 16 * 4;
constexpr int kSmem = 1024 + kWres + 2 * kWin + kTrans + kBars + kBred;
static_assert(kSmem <= 227 * 1024, "conv64 shared memory");
}  // namespace c64

__host__ __device__ __forceinline__ int c64_floor_div(int a, int b) {  // b > 0
    const int q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

// resident slot of tap (dh, dw) (window offsets dh·(W+2) + dw): pairs [(dh,−1), (dh,0)] in
// slots 2(dh+1), 2(dh+1)+1; singles (dh,+1) in slot 6 + 2(dh+1), its upper slot zero
__host__ __device__ __forceinline__ int c64_slot(int dh, int dw) {
    return dw == 1 ? 6 + 2 * (dh + 1) : 2 * (dh + 1) + dw + 1;
}

// 32 lanes × 32 columns plus the column after them (one wait)
__device__ __forceinline__ void tmem_ld33(uint32_t taddr, float* v, float& e) {
    uint32_t r[33];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x1.b32 {%32}, [%34];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31]), "=r"(r[32])
        : "r"(taddr), "r"(taddr + 32)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    e = __uint_as_float(r[32]);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void add_bf16x16(float* z, uint4 a, uint4 b) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        z[2 * e] += __uint_as_float(w[e] << 16);
        z[2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
    }
}

template <int MODE>
__global__ void __launch_bounds__(c64::kThreads, 1)
    conv64_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap bmap,
                  const Conv2Args a) {
    using namespace c64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sW = smem;
    uint8_t* sWin = sW + kWres;
    float* trans = reinterpret_cast<float*>(sWin + 2 * kWin);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(trans) + kTrans);
    uint64_t* wres_full = bars;
    uint64_t* wres_empty = bars + 1;
    uint64_t* wfull = bars + 2;   // [2] halo windows
    uint64_t* wempty = bars + 4;  // [2]
    uint64_t* tfull = bars + 6;   // [2] TMEM accumulators
    uint64_t* tempty = bars + 8;  // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);
    float* bred = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + kBars);  // [2][8 warps][16]

    constexpr int WTMA = kEpiWarps, WMMA = kEpiWarps + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int PH = a.H, PW = a.W;  // stride 1, pad 1: the output grid is the input grid
    const int PWp = PW + 2, PHp = PH + 1;
    const int ptiles = (a.B * PHp * PWp + kTileN - 1) / kTileN;
    const int64_t T = (int64_t)a.S * ptiles;
    const int t0 = (int)(T * blockIdx.x / gridDim.x), t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);

    // the zero upper halves of the single-tap groups (slots 7, 9, 11): written once
    for (int i = threadIdx.x; i < 3 * kBlk / 16; i += blockDim.x) {
        const int z = i / (kBlk / 16), o = i - z * (kBlk / 16);
        reinterpret_cast<uint4*>(sW + (7 + 2 * z) * kBlk)[o] = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(wres_full, 1);
        mbar_init(wres_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 1);
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps);
        }
        mbar_fence_init();
    }
    if (warp == WMMA) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == WTMA) {
        // ------------------------------------------------ TMA producer: resident W, windows
        if (lane == 0) {
            tma_prefetch_desc(&wmap);
            tma_prefetch_desc(&bmap);
            int cur_s = -1, seg = 0, tl = 0;
            for (int t = t0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                if (s != cur_s) {  // this sample's 9 tap blocks (after the previous sample's MMAs)
                    if (seg > 0) mbar_wait_role(wres_empty, (seg - 1) & 1);
                    mbar_arrive_expect_tx(wres_full, 9 * kBlk);
                    for (int tap = 0; tap < 9; ++tap) {
                        const int kh = tap / 3, kw = tap - 3 * kh;
                        const int dh = MODE == 0 ? kh - 1 : 1 - kh, dw = MODE == 0 ? kw - 1 : 1 - kw;
                        uint8_t* dst = sW + c64_slot(dh, dw) * kBlk;
                        if (MODE == 0)
                            tma_load_3d(&wmap, wres_full, dst, tap * 64, 0, s);  // [co][ci] K-major
                        else
                            tma_load_5d(&wmap, wres_full, dst, 0, tap, 0, 0, s);  // [co][ci]: MN-major A
                    }
                    cur_s = s;
                    ++seg;
                }
                const int ws = tl & 1;
                mbar_wait_role(&wempty[ws], ((tl >> 1) & 1) ^ 1);
                const int p0 = pt * kTileN;
                const int rs = c64_floor_div(p0 - PWp - 1, PWp), re = c64_floor_div(p0 + 256 + PWp, PWp);
                uint8_t* win = sWin + ws * kWin;
                mbar_arrive_expect_tx(&wfull[ws], (uint32_t)((re - rs + 1) * PWp * 128));
                for (int r = rs; r <= re; ++r) {
                    const int b = c64_floor_div(r, PHp), y = r - b * PHp;  // y == PH: separator (OOB: zeros)
                    tma_load_5d(&bmap, &wfull[ws], win + (r - rs) * PWp * 128, 0, -1, y, b, s);
                }
            }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        // ------------------------------------------------ MMA issuer: 6 groups × 4 K-steps per tile
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, 256, MODE == 1 ? 1 : 0, 0);
            int cur_s = -1, seg = 0, tl = 0;
            for (int t = t0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                if (s != cur_s) {
                    mbar_wait_role(wres_full, seg & 1);
                    cur_s = s;
                    ++seg;
                }
                const int buf = tl & 1;
                mbar_wait_role(&tempty[buf], ((tl >> 1) & 1) ^ 1);
                mbar_wait_role(&wfull[buf], (tl >> 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                const int p0 = pt * kTileN;
                const int wrow0 = p0 - c64_floor_div(p0 - PWp - 1, PWp) * PWp;  // window row of pixel p0
                const uint32_t winb = smem_u32(sWin + buf * kWin);
#pragma unroll
                for (int g = 0; g < 6; ++g) {
                    const int dh = (g < 3 ? g : g - 3) - 1, dw = g < 3 ? -1 : 1;  // the lower tap
                    const uint32_t aBase = smem_u32(sW + 2 * g * kBlk);
                    const uint32_t bBase = winb + (uint32_t)(wrow0 + dh * PWp + dw) * 128u;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = MODE == 0 ? sdesc_sw128(aBase + 32 * q, 16, 1024)
                                                      : sdesc_sw128(aBase + 2048 * q, kBlk, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 32 * q, 16, 1024);
                        mma_bf16(d, ad, bd, idesc, (g | q) != 0 ? 1u : 0u);
                    }
                }
                mma_commit(&wempty[buf]);
                mma_commit(&tfull[buf]);
                if (t + 1 < t1 && (t + 1) / ptiles != s) mma_commit(wres_empty);  // W free for the next sample
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue
        const int q = warp & 3, h = warp >> 2;
        const bool upper = q >= 2;
        const int cg = q & 1;             // channel group of 32
        const int pair = 1 + cg + 2 * h;  // named barrier of the lower/upper warp pair
        float* tr_self = trans + warp * 32 * kTransPitch;
        const float* tr_lo = trans + (upper ? warp - 2 : warp) * 32 * kTransPitch;
        const float* tr_up = trans + (upper ? warp : warp + 2) * 32 * kTransPitch;
        const int cl = upper ? 16 : 0;      // this thread's 16 channels within the group
        const int chq = cg * 32 + cl;       // … within the 64
        int tl = 0;
        for (int t = t0; t < t1; ++t, ++tl) {
            const int s = t / ptiles, pt = t - s * ptiles;
            const int buf = tl & 1;
            const int p0 = pt * kTileN;
            const int64_t so = (int64_t)s * a.out_stride_s;
            float bias16[16], bacc[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) bacc[k] = 0.0f;
            if (MODE == 0) {
                const float4* bs = reinterpret_cast<const float4*>(a.bias + (int64_t)s * a.CO + chq);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 b4 = __ldg(bs + k);
                    bias16[4 * k] = b4.x;
                    bias16[4 * k + 1] = b4.y;
                    bias16[4 * k + 2] = b4.z;
                    bias16[4 * k + 3] = b4.w;
                }
            }
            mbar_wait(&tfull[buf], (tl >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int i = 0; i < 4; ++i) {
                const int c = 4 * h + i;
                // the pass's pixel (thread = pixel after the transpose) and its operand rows: in
                // flight while the accumulator is read and transposed
                const int m = 32 * c + lane;
                const int pix = p0 + m;
                const int r = pix / PWp, cx = pix - r * PWp, b = r / PHp, y = r - b * PHp;
                const bool pv = m < kTileN && b < a.B && y < PH && cx >= 1 && cx <= PW;
                const int64_t rowoff = pv ? (((int64_t)b * PH + y) * PW + cx - 1) * 64 : 0;
                uint4 x0 = make_uint4(0u, 0u, 0u, 0u), x1 = x0;
                uint32_t mw = 0xFFFFFFFFu;
                const __nv_bfloat16* opnd = MODE == 0 ? a.res : a.addsrc;
                if (pv && opnd) {
                    const uint4* p = reinterpret_cast<const uint4*>(opnd + so + rowoff + chq);
                    x0 = MODE == 0 ? __ldg(p) : p[0];
                    x1 = MODE == 0 ? __ldg(p + 1) : p[1];
                }
                if (MODE == 1 && pv && a.mbits) mw = __ldg(a.mbits + ((so + rowoff + cg * 32) >> 5));
                float v[32], e = 0.0f;
                const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * 256 + 32 * c;
                if (upper && c < 7)
                    tmem_ld33(ta, v, e);
                else
                    tmem_ld32(ta, v);
                if (i == 3) {  // this warp's last TMEM read of the tile
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);
                }
                if (!upper) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) tr_self[j * kTransPitch + lane] = v[j];
                } else {  // upper column n + 1 holds pixel n
#pragma unroll
                    for (int j = 0; j < 31; ++j) tr_self[j * kTransPitch + lane] = v[j + 1];
                    tr_self[31 * kTransPitch + lane] = e;
                }
                named_bar(pair, 64);
                float z[16];
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    z[k] = tr_lo[lane * kTransPitch + cl + k] + tr_up[lane * kTransPitch + cl + k];
                named_bar(pair, 64);  // both halves read before the next chunk overwrites them
                if (!pv) continue;
                if (MODE == 0) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) z[k] += bias16[k];
                    if (a.res) add_bf16x16(z, x0, x1);
                    if (a.relu) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) z[k] = fmaxf(z[k], 0.0f);
                    }
                } else {
                    if (a.addsrc) add_bf16x16(z, x0, x1);
                    const uint32_t mb = mw >> cl;
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (!((mb >> k) & 1u)) z[k] = 0.0f;
#pragma unroll
                    for (int k = 0; k < 16; ++k) bacc[k] += z[k];
                }
                uint32_t pk[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) pk[k] = pack_bf16x2(z[2 * k], z[2 * k + 1]);
                uint4* op = reinterpret_cast<uint4*>(a.out + so + rowoff + chq);
                op[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                op[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                if (MODE == 0 && a.mbits_out) {  // bits of the stored bf16 values (> 0), 16 per thread
                    uint32_t bits = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t lo = pk[k] & 0xFFFFu, hi = pk[k] >> 16;
                        bits |= (uint32_t)((lo & 0x7FFFu) != 0 && (lo & 0x8000u) == 0) << (2 * k);
                        bits |= (uint32_t)((hi & 0x7FFFu) != 0 && (hi & 0x8000u) == 0) << (2 * k + 1);
                    }
                    reinterpret_cast<uint16_t*>(a.mbits_out)[((so + rowoff + cg * 32) >> 4) + (upper ? 1 : 0)] =
                        (uint16_t)bits;
                }
            }
            if (MODE == 1 && a.bpart) {  // Σ over the tile's pixels per channel, fixed order
#pragma unroll
                for (int k = 0; k < 16; ++k) tr_self[lane * kTransPitch + k] = bacc[k];
                __syncwarp();
                float sum = 0.0f;
                if (lane < 16) {
#pragma unroll 8
                    for (int r = 0; r < 32; ++r) sum += tr_self[r * kTransPitch + lane];
                }
                __syncwarp();
                float* red = bred + (tl & 1) * kEpiWarps * 16;
                if (lane < 16) red[warp * 16 + lane] = sum;
                named_bar(5, kEpiWarps * 32);
                if (h == 0 && lane < 16)
                    a.bpart[(int64_t)s * a.bpart_stride_s + (int64_t)pt * a.C + chq + lane] =
                        red[warp * 16 + lane] + red[(warp + 4) * 16 + lane];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int conv64_ok(int H, int W) {  // the padded window of a 255-pixel tile fits one window stage
    const int PWp = W + 2;
    const int rows = (256 + 2 * PWp + 1 + PWp - 1) / PWp + 1;
    return H >= 1 && rows * PWp * 128 <= c64::kWin ? 1 : 0;
}

int conv64_parts(const Conv2Args& a) { return (a.B * (a.H + 1) * (a.W + 2) + c64::kTileN - 1) / c64::kTileN; }

template <int MODE>
static void launch_conv64(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(conv64_kernel<MODE>), c64::kSmem);
    const int64_t T = (int64_t)a.S * conv64_parts(a);
    conv64_kernel<MODE><<<(int)std::min<int64_t>(T, kNumSMs), c64::kThreads, c64::kSmem, st>>>(wmap, bmap, a);
}

void launch_conv64_fwd(const CUtensorMap& wmap, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv64<0>(wmap, bmap, a, st);
}
void launch_conv64_dgrad(const CUtensorMap& wmapT, const CUtensorMap& bmap, const Conv2Args& a, cudaStream_t st) {
    launch_conv64<1>(wmapT, bmap, a, st);
}

}  // namespace bnn
