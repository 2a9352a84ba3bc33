// kernels_stem.cu — the ResNet stem (3 → 64 channels, 3×3, stride 1) forward on tcgen05, K3
// (PAPER.md:160):  Y[p][co] = ReLU( Σ_{kh,kw,ci} X[p ⊕ (kh−1, kw−1)][ci] · W_s[co][kh,kw,ci] + b_s[co] ).
//
// The input has 8 (padded) channels: 16 bytes per pixel. With SWIZZLE_NONE K-major operands an
// MMA's K = 16 is two 8-channel core-matrix columns whose distance is the descriptor's leading
// byte offset — any multiple of 16 B. So one MMA takes TWO taps: A = the halo window of the padded
// pixel stream at tap a's offset with LBO = (offset_b − offset_a)·16 B, B = the two taps' 8 × 64
// weight blocks with LBO = their distance. 9 taps = 5 MMAs (M = 128 pixels, N = 64, the last pair
// with a zero block) per 128-pixel tile, every tap accumulating into the same TMEM lane = pixel:
// no shifted sums, no transposes; the epilogue is thread = pixel over its 64 channels (+ bias,
// ReLU, RN-bf16, ReLU bitmask, 32-byte stores). W_s of every sample of the chunk (10 × 1 KB core-
// matrix blocks each) is staged in shared memory once per CTA from the layer's W scratch slot.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_conv.cuh"
#include "tc_ptx.cuh"

namespace bnn {

using namespace ptx;

namespace stem {
constexpr int kGroups = 4;                     // epilogue groups of 4 warps (one per TMEM lane quarter), tiles round-robin
constexpr int kEpiWarps = 4 * kGroups;
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int kTile = 128;                    // padded-stream positions per tile (all 128 rows are outputs)
constexpr int kWBlk = 1024;                   // one tap: 8 co-groups × (8 rows × 16 B) core matrices
constexpr int kWSample = 10 * kWBlk;          // 9 taps + a zero block
constexpr int kSlots = 2;                     // a CTA's contiguous tile range spans ≤ 2 samples
constexpr int kNWin = 8;
constexpr int kWin = 320 * 16;                // ≤ 320 padded pixels (7 rows of 40) × 16 B
constexpr int kSmem = 1024 + kSlots * kWSample + kNWin * kWin + 256;
}  // namespace stem

// UMMA shared-memory descriptor, no swizzle (layout type 0): core matrices of 8 rows × 16 B,
// `lbo` between K-adjacent core matrices, `sbo` between M/N-adjacent ones
__device__ __forceinline__ uint64_t sdesc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}

__host__ __device__ __forceinline__ int stem_pitch(int W) { return (W + 2 + 7) / 8 * 8; }

__device__ __forceinline__ int stem_floor_div(int a, int b) {
    const int q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

__device__ __forceinline__ void st256s(void* p, const uint32_t* r) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__global__ void __launch_bounds__(stem::kThreads, 1)
    stem_fwd_kernel(const __grid_constant__ StemRowMaps xmaps, const Conv2Args a) {
    using namespace stem;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sW = smem;                               // [s][10 taps][8 co-groups][8 × 16 B]
    uint8_t* sWin = sW + kSlots * kWSample;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sWin + kNWin * kWin);
    uint64_t* wfull = bars;                  // [kNWin]
    uint64_t* wempty = bars + kNWin;         // [kNWin]
    uint64_t* tfull = bars + 2 * kNWin;      // [kGroups] TMEM accumulators of 64 columns
    uint64_t* tempty = tfull + kGroups;      // [kGroups]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + kGroups);
    constexpr int WTMA = kEpiWarps, WMMA = kEpiWarps + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // padded rows of round_up(W + 2, 8) pixels = a multiple of 128 B (TMA destinations stay 128-B aligned)
    const int PH = a.H, PW = a.W, PWp = stem_pitch(PW), PHp = PH + 1;
    const int ptiles = (a.B * PHp * PWp + kTile - 1) / kTile;
    const int64_t T = (int64_t)a.S * ptiles;
    const int t0 = (int)(T * blockIdx.x / gridDim.x), t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);
    const int s_lo = t0 / ptiles, s_hi = (t1 - 1) / ptiles;

    // W_s of this CTA's samples into core-matrix order: element (co, tap, ci) of sample s at
    // s·kWSample + tap·1024 + (co / 8)·128 + (co % 8)·16 + ci·2 (tap 9: zeros)
    for (int i = threadIdx.x; i < (s_hi - s_lo + 1) * 10 * 64; i += blockDim.x) {
        const int sl = i / 640, rem = i - sl * 640, tap = rem / 64, co = rem - tap * 64;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (tap < 9) v = *reinterpret_cast<const uint4*>(a.wsrc + ((int64_t)(s_lo + sl) * 64 + co) * a.K_pad + tap * 8);
        *reinterpret_cast<uint4*>(sW + sl * kWSample + tap * kWBlk + (co >> 3) * 128 + (co & 7) * 16) = v;
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kNWin; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 1);
        }
        for (int i = 0; i < kGroups; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_fence_init();
    }
    if (warp == WMMA) tmem_alloc(tslot, 64 * kGroups);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == WTMA) {
        if (lane == 0) {

            for (int t = t0, tl = 0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                const int ws = tl % kNWin;
                mbar_wait_role(&wempty[ws], ((tl / kNWin) & 1) ^ 1);
                const int p0 = pt * kTile;
                const int rs = stem_floor_div(p0 - PWp - 1, PWp), re = stem_floor_div(p0 + kTile + PWp, PWp);
                mbar_arrive_expect_tx(&wfull[ws], (uint32_t)((re - rs + 1) * PWp * 16));
                for (int r = rs; r <= re;) {  // one op per run of padded rows inside one image
                    const int b = stem_floor_div(r, PHp), y = r - b * PHp;  // y == PH, b ∉ [0, B): zeros
                    const int run = min(min(re, b * PHp + PH) - r + 1, min(8, PH));
                    tma_load_5d(&xmaps.x[run - 1], &wfull[ws], sWin + ws * kWin + (r - rs) * PWp * 16, 0, -1, y, b,
                                a.src_stride_s == 0 ? 0 : s);
                    r += run;
                }
            }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, 64, 0, 0);
            for (int t = t0, tl = 0; t < t1; ++t, ++tl) {
                const int s = t / ptiles, pt = t - s * ptiles;
                const int buf = tl % kGroups, ws = tl % kNWin;
                mbar_wait_role(&tempty[buf], ((tl / kGroups) & 1) ^ 1);
                mbar_wait_role(&wfull[ws], (tl / kNWin) & 1);
                tc_fence_after();
                const int p0 = pt * kTile;
                const int wrow0 = p0 - stem_floor_div(p0 - PWp - 1, PWp) * PWp;  // window position of p0
                const uint32_t winb = smem_u32(sWin + ws * kWin);
                const uint32_t wb = smem_u32(sW + (s - s_lo) * kWSample);
#pragma unroll
                for (int pr = 0; pr < 5; ++pr) {  // taps (2pr, 2pr+1); pair 4 = (8, zero block)
                    const int ta = 2 * pr, tb = 2 * pr + 1;
                    const int oa = (ta / 3 - 1) * PWp + (ta % 3 - 1);
                    const int ob = tb < 9 ? (tb / 3 - 1) * PWp + (tb % 3 - 1) : oa;  // zero block: re-read tap a
                    const uint64_t ad = sdesc_none(winb + (uint32_t)(wrow0 + oa) * 16u, (uint32_t)(ob - oa) * 16u, 128);
                    const uint64_t bd = sdesc_none(wb + ta * kWBlk, kWBlk, 128);
                    mma_bf16(tmem + buf * 64, ad, bd, idesc, pr != 0 ? 1u : 0u);
                }
                mma_commit(&wempty[ws]);
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else {
        // epilogue: group g = warp / 4 takes the tiles of TMEM buffer g; warp = lane quarter q
        // (pixels 32q … 32q + 31), thread = pixel with its 64 channels (two passes of 32)
        const int g = warp >> 2, q = warp & 3;
        const int m = 32 * q + lane;
        for (int t = t0 + g, tl = g; t < t1; t += kGroups, tl += kGroups) {
            const int s = t / ptiles, pt = t - s * ptiles;
            const int pix = pt * kTile + m;
            const int r = pix / PWp, cx = pix - r * PWp, b = r / PHp, y = r - b * PHp;
            const bool pv = b < a.B && y < PH && cx >= 1 && cx <= PW;
            const int64_t ro = pv ? (((int64_t)b * PH + y) * PW + cx - 1) * 64 : 0;
            const int64_t so = (int64_t)s * a.out_stride_s;
            epi_wait(&tfull[g], (tl / kGroups) & 1);
            tc_fence_after();
            const float4* bs = reinterpret_cast<const float4*>(a.bias + (int64_t)s * a.CO);
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {  // two passes of 32 channels (96-register budget of 18 warps)
                float v[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + g * 64 + c0, v);
                if (c0 == 32) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[g]);
                }
                if (!pv) continue;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float4 b4 = __ldg(bs + c0 / 4 + k);
                    v[4 * k] = fmaxf(v[4 * k] + b4.x, 0.0f);
                    v[4 * k + 1] = fmaxf(v[4 * k + 1] + b4.y, 0.0f);
                    v[4 * k + 2] = fmaxf(v[4 * k + 2] + b4.z, 0.0f);
                    v[4 * k + 3] = fmaxf(v[4 * k + 3] + b4.w, 0.0f);
                }
                uint32_t pk[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) pk[k] = pack_bf16x2(v[2 * k], v[2 * k + 1]);
                st256s(a.out + so + ro + c0, pk);
                st256s(a.out + so + ro + c0 + 16, pk + 8);
                if (a.mbits_out) {  // bit j = stored bf16 of channel c0 + j > 0 (no negative values after the ReLU)
                    uint32_t bits = 0;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const uint32_t cb = ((pk[k] & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x80008000u;
                        bits |= (((cb >> 15) & 1u) | (cb >> 30)) << (2 * k);
                    }
                    a.mbits_out[(so + ro + c0) >> 5] = bits;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 64 * kGroups);
    }
}

int stem_fwd_ok(const Conv2Args& a) {  // 3×3 stride-1 pad-1, 8 padded input channels, 64 outputs, ReLU, no residual
    const int PWp = stem_pitch(a.W);
    const int rows = (stem::kTile + 3 * PWp) / PWp + 1;
    return a.k == 3 && a.stride == 1 && a.pad == 1 && a.C_pad == 8 && a.C <= 8 && a.CO == 64 && a.relu && !a.res &&
                   a.K_pad >= 72 && a.wsrc && rows * PWp * 16 <= stem::kWin
               ? 1
               : 0;
}

int stem_row_pitch(int W) { return stem_pitch(W); }

void launch_stem_fwd(const StemRowMaps& xmaps, const Conv2Args& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(stem_fwd_kernel), stem::kSmem);
    const int ptiles = (a.B * (a.H + 1) * stem_pitch(a.W) + stem::kTile - 1) / stem::kTile;
    const int64_t T = (int64_t)a.S * ptiles;
    stem_fwd_kernel<<<(int)std::min<int64_t>(T, kNumSMs), stem::kThreads, stem::kSmem, st>>>(xmaps, a);
    if (getenv("BNN_DEBUG_SYNC")) {
        cudaError_t e1 = cudaGetLastError(), e2 = cudaStreamSynchronize(st);
        fprintf(stderr, "stem_fwd_kernel: launch %s, sync %s (smem %d, threads %d)\n", cudaGetErrorString(e1),
                cudaGetErrorString(e2), stem::kSmem, stem::kThreads);
    }
}

}  // namespace bnn
