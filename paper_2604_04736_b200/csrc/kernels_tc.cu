// kernels_tc.cu — BF16 tensor-core sampled-layer kernels for sm_100a.
//
// K2 (fwd):   Z_s = X_s · W_sᵀ + b_s, ReLU                       PAPER.md:160 (Alg. 1 l.7)
// K4 (dgrad): dX_s = (G_s · W_s) ⊙ 1[X_s > 0]                    PAPER.md:165 (Alg. 1 l.12)
// K5 (wgrad): dW_s = G_sᵀ · X_s;  acc_μ += dW_s,  acc_ρ += dW_s ⊙ ε_s over the CTA's samples
//             (north_star subsystem (3); reading R20: sigmoid(ρ) is applied once in K8)
//
// The sampled weight tile W_s = RN_bf16(fma(σ, ε_s, μ)) is produced on chip by eight
// generator warps straight into the UMMA canonical SWIZZLE_128B layout in shared memory
// (north_star subsystem (2)); it is never written to global memory. Activations and
// gradients are TMA-loaded; one elected thread issues tcgen05.mma (M=128, K=16 steps) with
// the fp32 accumulator in TMEM; the epilogue reads TMEM with tcgen05.ld.
//
// Operand orientation (tcgen05 computes D[M×N] = A[M×K]·B[N×K]ᵀ):
//   fwd   : M = output feature n, N = batch b, K = fan-in k. A = W_s tile, K-major (as
//           generated); B = X_s [b][k], K-major (TMA box 64 k × 256 b).
//   dgrad : M = input feature k, N = batch b, K = output feature n. A = W_sᵀ: the same
//           generated rows of W_s, stored MN-major (k contiguous); B = G_s [b][n], K-major.
//   wgrad : M = n, N = k (64-wide tiles), K = batch b. A = G_sᵀ, MN-major; B = X_s, MN-major.
#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "kernels_tc.cuh"
#include "tc_ptx.cuh"

namespace bnn {

using namespace ptx;

// ============================================================================ K2 / K4
namespace gen {
constexpr int kGenWarps = 8;  // 16 was measured: issue-active 64 -> 76 %, no faster (56 regs)
constexpr int kItems = kGenWarps == 16 ? 4 : 8;  // 4-element items per thread per k-block
constexpr int kThreads = (kGenWarps + 1) * 32;  // + one control warp (TMEM alloc, MMA issue)
constexpr int kAStage = 128 * 64 * 2;           // 16 KB generated W tile
constexpr int kBStage = 256 * 64 * 2;           // 32 KB activation/gradient tile
constexpr int smem_bytes(int stages) { return 1024 + stages * (kAStage + kBStage) + 256 + 128 * 4; }
}  // namespace gen

__device__ __forceinline__ void load_mu_sigma4(const SampledLayer& L, int64_t i, int kvalid,
                                               bool vec, float4& m, float4& sg) {
    if (vec && kvalid >= 4) {
        m = __ldg(reinterpret_cast<const float4*>(L.mu + i));
        sg = __ldg(reinterpret_cast<const float4*>(L.sigma + i));
    } else {
        float mm[4] = {0.f, 0.f, 0.f, 0.f}, ss[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < 4 && j < kvalid; ++j) {
            mm[j] = __ldg(L.mu + i + j);
            ss[j] = __ldg(L.sigma + i + j);
        }
        m = make_float4(mm[0], mm[1], mm[2], mm[3]);
        sg = make_float4(ss[0], ss[1], ss[2], ss[3]);
    }
}

// W_s[n][k .. k+3] as two packed bf16x2 words (zero outside the tensor). Checked path,
// used only for edge tiles.
__device__ __forceinline__ uint2 gen_w4(const SampledLayer& L, const SampleKeys& kk, uint32_t sg,
                                        int n, int k, bool vec) {
    if (n >= L.N || k >= L.K) return make_uint2(0u, 0u);
    const int kvalid = L.K - k;
    const int64_t i = L.off_w + (int64_t)n * L.K + k;
    float4 m, s;
    load_mu_sigma4(L, i, kvalid, vec, m, s);
    const float4 e = eps4(kk.key, kk.step, sg, L.t_w, (uint32_t)n, (uint32_t)(k >> 2));
    float w0 = __fmaf_rn(s.x, e.x, m.x), w1 = __fmaf_rn(s.y, e.y, m.y);
    float w2 = __fmaf_rn(s.z, e.z, m.z), w3 = __fmaf_rn(s.w, e.w, m.w);
    if (kvalid < 4) {
        w1 = kvalid > 1 ? w1 : 0.f;
        w2 = kvalid > 2 ? w2 : 0.f;
        w3 = 0.f;
    }
    return make_uint2(pack_bf16x2(w0, w1), pack_bf16x2(w2, w3));
}

// Fast path: interior tile, 16-byte aligned μ/σ rows, no bounds checks.
__device__ __forceinline__ uint2 gen_w4_fast(const float* __restrict__ mu,
                                             const float* __restrict__ sigma, const EpsKey& key,
                                             uint32_t step, uint32_t w3, uint32_t n, uint32_t cq) {
    const float4 m = __ldg(reinterpret_cast<const float4*>(mu));
    const float4 s = __ldg(reinterpret_cast<const float4*>(sigma));
    const uint4 y = philox10(make_uint4(cq, n, w3, step), key);
    const float R0 = bm_radius(y.x);
    const float2 cs0 = bm_sincos(y.y);
    const float R1 = bm_radius(y.z);
    const float2 cs1 = bm_sincos(y.w);
    const float w0 = __fmaf_rn(s.x, __fmul_rn(R0, cs0.x), m.x);
    const float w1 = __fmaf_rn(s.y, __fmul_rn(R0, cs0.y), m.y);
    const float w2 = __fmaf_rn(s.z, __fmul_rn(R1, cs1.x), m.z);
    const float w3v = __fmaf_rn(s.w, __fmul_rn(R1, cs1.y), m.w);
    return make_uint2(pack_bf16x2(w0, w1), pack_bf16x2(w2, w3v));
}

__device__ __forceinline__ void sts64(uint32_t addr, uint2 v) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}

template <int MODE, int STAGES>
__global__ void __launch_bounds__(gen::kThreads, 2)
    gen_gemm_kernel(const __grid_constant__ CUtensorMap tmB, const TcGenArgs a) {
    using namespace gen;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment as an offset into the __shared__ array: the pointer keeps the shared
    // address space, so plain loads/stores through it compile to LDS/STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * kBStage);
    uint64_t* full_gen = bars;
    uint64_t* full_tma = bars + STAGES;
    uint64_t* empty = bars + 2 * STAGES;
    uint64_t* tfull = bars + 3 * STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 1);
    float* sbias = reinterpret_cast<float*>(bars + 32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int m0 = blockIdx.x * 128, s = blockIdx.y, b0 = blockIdx.z * 256;
    const uint32_t sg = a.kk.s0 + s;
    const SampledLayer& L = a.L;

    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full_gen[i], kGenWarps);
            mbar_init(&full_tma[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_fence_init();
        tma_prefetch_desc(&tmB);
    }
    if (warp == kGenWarps) tmem_alloc(tslot, 256);
    if (MODE == 0 && tid < 128) {
        const int n = m0 + tid;
        sbias[tid] = n < L.N ? __fmaf_rn(L.sigma[L.off_b + n],
                                         eps1(a.kk.key, a.kk.step, sg, L.t_b, 0u, (uint32_t)n),
                                         L.mu[L.off_b + n])
                             : 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int nkb = (a.R + 63) / 64;

    if (warp == kGenWarps) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, a.nb, MODE == 1 ? 1 : 0, 0);
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait_suspend(&full_gen[st], ph);
                mbar_wait_suspend(&full_tma[st], ph);
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
    } else {
        // ------------------------------------------------ generator warps
        // Thread → item mapping (constant per thread; `it` advances the row):
        //   fwd  : row = it*rstep + (tid>>4) (output feature n), quad kq = tid&15 of the 64 k
        //   dgrad: row = it*rstep + (tid>>5) (output feature n = the MMA K dim), quad mq = tid&31
        //          of the 128 k of this M tile (two 64-wide MN blocks)
        // The 128B-swizzle chunk depends on row&7, which is constant per thread.
        const int rsub = MODE == 0 ? (tid >> 4) : (tid >> 5);
        const int qd = MODE == 0 ? (tid & 15) : (tid & 31);
        const int rstep = MODE == 0 ? kGenWarps * 2 : kGenWarps;
        const uint32_t soff0 =
            MODE == 0 ? rsub * 128 + ((((qd >> 1) ^ (rsub & 7))) << 4) + ((qd & 1) << 3)
                      : (qd >> 4) * 8192 + rsub * 128 + (((((qd & 15) >> 1) ^ (rsub & 7))) << 4) +
                            ((qd & 1) << 3);
        const uint32_t sstep = rstep * 128;
        const bool vec = a.vec_ok != 0;
        const uint32_t w3 = (L.t_w << 20) | sg;
        const bool m_full = MODE == 0 ? (m0 + 128 <= L.N) : (m0 + 128 <= L.K);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            if (tid == 0) {
                mbar_arrive_expect_tx(&full_tma[st], kBStage);
                tma_load_3d(&tmB, &full_tma[st], sB + st * kBStage, kb * 64, b0,
                            a.b_shared ? 0 : s);
            }
            const uint32_t tileA = smem_u32(sA + st * kAStage) + soff0;
            const bool full = vec && m_full &&
                              (MODE == 0 ? (kb * 64 + 64 <= L.K) : (kb * 64 + 64 <= L.N));
            if (full) {
                // n, k of item 0; item `it` adds rstep rows
                const int n0 = MODE == 0 ? m0 + rsub : kb * 64 + rsub;
                const int k0 = MODE == 0 ? kb * 64 + 4 * qd : m0 + 4 * qd;
                const int64_t e0 = L.off_w + (int64_t)n0 * L.K + k0;
                const float* mup = L.mu + e0;
                const float* sgp = L.sigma + e0;
                const int64_t estep = (int64_t)rstep * L.K;
                if (a.mu_only) {  // MC dropout: RN_bf16(fma(0, ε, μ)) = RN_bf16(μ)
#pragma unroll 4
                    for (int it = 0; it < kItems; ++it) {
                        const float4 m = __ldg(reinterpret_cast<const float4*>(mup + it * estep));
                        sts64(tileA + it * sstep, make_uint2(pack_bf16x2(m.x, m.y), pack_bf16x2(m.z, m.w)));
                    }
                } else {
#pragma unroll 4
                    for (int it = 0; it < kItems; ++it) {
                        const uint2 w = gen_w4_fast(mup + it * estep, sgp + it * estep, a.kk.key,
                                                    a.kk.step, w3, (uint32_t)(n0 + it * rstep),
                                                    (uint32_t)(k0 >> 2));
                        sts64(tileA + it * sstep, w);
                    }
                }
            } else if (MODE == 0 && vec && m_full && ((L.K - kb * 64) & 3) == 0) {
                // forward, last k-block of a fan-in that is not a multiple of 64 (784 = 12·64 + 16):
                // the valid quads are spread over all threads (the fixed mapping above would leave
                // 3/4 of the lanes idle for a 16-column block), the rest of the tile is zeroed
                const int nq = (L.K - kb * 64) >> 2;  // valid 4-column quads per row
                const uint32_t tile0 = smem_u32(sA + st * kAStage);
                for (int i = tid; i < 128 * nq; i += kGenWarps * 32) {
                    const int r = i / nq, qq = i - r * nq;
                    const int64_t e = L.off_w + (int64_t)(m0 + r) * L.K + kb * 64 + 4 * qq;
                    const uint2 w = gen_w4_fast(L.mu + e, L.sigma + e, a.kk.key, a.kk.step, w3,
                                                (uint32_t)(m0 + r), (uint32_t)((kb * 64 >> 2) + qq));
                    sts64(tile0 + r * 128 + ((((qq >> 1) ^ (r & 7))) << 4) + ((qq & 1) << 3), w);
                }
                for (int i = tid; i < 128 * (16 - nq); i += kGenWarps * 32) {
                    const int r = i / (16 - nq), qq = nq + (i - r * (16 - nq));
                    sts64(tile0 + r * 128 + ((((qq >> 1) ^ (r & 7))) << 4) + ((qq & 1) << 3), make_uint2(0u, 0u));
                }
            } else {
#pragma unroll 1
                for (int it = 0; it < kItems; ++it) {
                    const int n = MODE == 0 ? m0 + rsub + it * rstep : kb * 64 + rsub + it * rstep;
                    const int k = MODE == 0 ? kb * 64 + 4 * qd : m0 + 4 * qd;
                    sts64(tileA + it * sstep, gen_w4(L, a.kk, sg, n, k, vec));
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_gen[st]);
        }
        // ------------------------------------------------ epilogue
        const int q = warp & 3, h = warp >> 2;
        const int row = 32 * q + lane, m = m0 + row;
        const int nchunks = (a.nb + 15) / 16;
        constexpr int kCStep = kGenWarps / 4;
        // dgrad: the ReLU-mask rows of a chunk are loaded one chunk ahead (the first before the
        // accumulator wait), so their latency overlaps the MMA and the previous chunk
        uint16_t mnext[16];
        auto load_mask = [&](int c) {
            const int bc0 = b0 + c * 16;
            const int nvalid = min(16, a.B - bc0);
            if (MODE == 1 && a.mask && m < a.M && nvalid > 0 && c < nchunks) {
                const uint16_t* mk = reinterpret_cast<const uint16_t*>(a.mask) + s * a.mask_stride_s +
                                     (int64_t)bc0 * a.ldm + m;
#pragma unroll
                for (int j = 0; j < 16; ++j) mnext[j] = j < nvalid ? __ldg(mk + (int64_t)j * a.ldm) : 0;
            }
        };
        if (MODE == 1) load_mask(h);
        mbar_wait_suspend(tfull, 0);
        tc_fence_after();
        const float bias = MODE == 0 ? sbias[row] : 0.0f;
        for (int c = h; c < nchunks; c += kCStep) {
            const int bc0 = b0 + c * 16;
            const int nvalid = min(16, a.B - bc0);
            const bool live = m < a.M && nvalid > 0;
            uint16_t mraw[16];
            if (MODE == 1) {
#pragma unroll
                for (int j = 0; j < 16; ++j) mraw[j] = mnext[j];
                load_mask(c + kCStep);
            }
            float v[16];
            __syncwarp();
            tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + c * 16, v);
            if (!live) continue;
            if (MODE == 0) {
                if (a.out_f32) {
                    float* o = reinterpret_cast<float*>(a.out) + s * a.out_stride_s + (int64_t)bc0 * a.ldo + m;
                    // res_f32: + the fp32 residual stream (the ViT's X + proj(·), X + fc2(·))
                    float rv[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) rv[j] = 0.0f;
                    if (a.res_f32) {  // all 16 loads issued before any store (o and r may not alias)
                        const float* r = a.res_f32 + s * a.out_stride_s + (int64_t)bc0 * a.ldo + m;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (j < nvalid) rv[j] = __ldg(r + (int64_t)j * a.ldo);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < nvalid) o[(int64_t)j * a.ldo] = v[j] + bias + rv[j];
                } else {
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(a.out) + s * a.out_stride_s +
                                       (int64_t)bc0 * a.ldo + m;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (j < nvalid) {
                            float z = v[j] + bias;
                            if (a.relu) z = fmaxf(z, 0.0f);
                            if (a.drop.on)  // MC dropout after the hidden activation (R25)
                                z = dropout_keep(a.kk.key, a.kk.step, sg, (uint32_t)a.drop.layer,
                                                 (uint32_t)(a.drop.b_off + bc0 + j), (uint32_t)m, a.drop.p24)
                                        ? z * a.drop.inv_keep : 0.0f;
                            o[(int64_t)j * a.ldo] = __float2bfloat16_rn(z);
                        }
                    }
                }
            } else {
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(a.out) + s * a.out_stride_s +
                                   (int64_t)bc0 * a.ldo + m;
                float* of = reinterpret_cast<float*>(a.out) + s * a.out_stride_s + (int64_t)bc0 * a.ldo + m;
                float part = 0.0f;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j < nvalid) {
                        // ReLU mask of the layer input: bf16 > 0 ⟺ sign bit clear and ≠ 0
                        // (MC dropout: a dropped unit is stored as 0, a kept one carries 1/(1 − p))
                        const float g =
                            (!a.mask || (mraw[j] != 0 && (mraw[j] & 0x8000u) == 0))
                                ? (a.drop.on ? v[j] * a.drop.inv_keep : v[j]) : 0.0f;
                        part += g;
                        // out_f32: the ViT's dgrad outputs feed fp32 LayerNorm / GELU / attention backward
                        if (a.out_f32)
                            of[(int64_t)j * a.ldo] = g;
                        else
                            o[(int64_t)j * a.ldo] = __float2bfloat16_rn(g);
                    }
                }
                // fp32 partial column sum over this 16-row chunk: the bias gradient source
                if (a.dbpart) a.dbpart[s * a.dbpart_stride_s + (int64_t)(bc0 >> 4) * a.M + m] = part;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kGenWarps) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// ============================================================================ K2 / K4, W-stationary
// For layers with many batch rows per sample (the ViT's token rows: 33 tiles of 256 per sample)
// the kernel above regenerates the same W_s tile once per 256-row tile. Here a CTA owns
// (m-tile, sample, a chunk of row tiles): its generator warps form the whole W_s tile ONCE into
// resident shared memory (R ≤ 256: ≤ 4 k-blocks, 64 KB), then the CTA streams the chunk's row
// tiles through it — a TMA warp fills a ring of activation / gradient stages, the MMA thread
// accumulates each row tile in one of two TMEM buffers, and the generator warps, done
// generating, run the epilogue of tile i while tile i+1 is multiplied. W_s is still never in HBM
// and ε is drawn once per (element, sample, chunk) instead of once per (element, sample, tile).
// Epilogue features: fwd — fp32 out (+ bias, + res_f32) or bf16 (+ bias, ReLU); dgrad — fp32 or
// bf16 out, no activation mask (the ViT's projections).
// Two shapes: NB = 256 rows per tile with R ≤ 256 (4 resident k-blocks, 3 row stages), and
// NB = 128 with R ≤ 768 (12 resident k-blocks = 192 KB, 2 row stages of 16 KB; N = 128 MMAs).
namespace gws {
constexpr int kThreads = (gen::kGenWarps + 2) * 32;  // + MMA warp + TMA warp
template <int NB>
struct Shape {
    static constexpr int kMaxKb = NB == 256 ? 4 : 12;
    static constexpr int kBStages = NB == 256 ? 3 : 2;
    static constexpr int kBStage = NB * 64 * 2;
    static constexpr int kSmem = 1024 + kMaxKb * gen::kAStage + kBStages * kBStage + 256 + 128 * 4;
};
static_assert(Shape<128>::kSmem <= 227 * 1024, "W-stationary NB=128 shared memory");
}  // namespace gws

template <int MODE, int NB>
__global__ void __launch_bounds__(gws::kThreads, 1)
    gen_gemm_ws_kernel(const __grid_constant__ CUtensorMap tmB, const TcGenArgs a, int tiles_per) {
    using namespace gen;
    constexpr int kBStages = gws::Shape<NB>::kBStages, kMaxKb = gws::Shape<NB>::kMaxKb;
    constexpr int kBStage = gws::Shape<NB>::kBStage;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                                   // resident W_s k-blocks
    uint8_t* sB = smem + kMaxKb * kAStage;                 // ring of row-tile k-blocks
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kBStages * kBStage);
    uint64_t* wfull = bars;                                // [kMaxKb] W_s k-block formed
    uint64_t* full = bars + kMaxKb;                        // [kBStages]
    uint64_t* empty = full + kBStages;                     // [kBStages]
    uint64_t* tfull = empty + kBStages;                    // [2]
    uint64_t* tempty = tfull + 2;                          // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sbias = reinterpret_cast<float*>(bars + 32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int m0 = blockIdx.x * 128, s = blockIdx.y;
    const int ntiles_b = (a.B + NB - 1) / NB;
    const int t0 = blockIdx.z * tiles_per, t1 = min(ntiles_b, t0 + tiles_per);
    const uint32_t sg = a.kk.s0 + s;
    const SampledLayer& L = a.L;
    const int nkb = (a.R + 63) / 64;
    const int WMMA = kGenWarps, WTMA = kGenWarps + 1;

    if (tid == 0) {
        for (int i = 0; i < kMaxKb; ++i) mbar_init(&wfull[i], kGenWarps);
        for (int i = 0; i < kBStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kGenWarps);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmB);
    }
    if (warp == WMMA) tmem_alloc(tslot, 2 * NB);
    if (MODE == 0 && tid < 128) {
        const int n = m0 + tid;
        sbias[tid] = n < L.N ? __fmaf_rn(L.sigma[L.off_b + n], eps1(a.kk.key, a.kk.step, sg, L.t_b, 0u, (uint32_t)n),
                                         L.mu[L.off_b + n])
                             : 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == WTMA) {
        // ------------------------------------------------ TMA: row tiles × k-blocks through the ring
        if (lane == 0) {
            int it = 0;
            for (int bt = t0; bt < t1; ++bt)
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kBStages;
                    mbar_wait_role(&empty[st], ((it / kBStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[st], kBStage);
                    tma_load_3d(&tmB, &full[st], sB + st * kBStage, kb * 64, bt * NB, a.b_shared ? 0 : s);
                }
        }
        __syncwarp();
    } else if (warp == WMMA) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, a.nb, MODE == 1 ? 1 : 0, 0);
            for (int kb = 0; kb < nkb; ++kb) mbar_wait_role(&wfull[kb], 0);
            int it = 0, tl = 0;
            for (int bt = t0; bt < t1; ++bt, ++tl) {
                const int buf = tl & 1;
                mbar_wait_role(&tempty[buf], ((tl >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * NB;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kBStages;
                    mbar_wait_role(&full[st], (it / kBStages) & 1);
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + kb * kAStage);
                    const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = MODE == 0 ? sdesc_sw128(aBase + 32 * q, 16, 1024)
                                                      : sdesc_sw128(aBase + 2048 * q, 8192, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 32 * q, 16, 1024);
                        mma_bf16(d, ad, bd, idesc, (kb | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ generators: the resident W_s tile
        const int rsub = MODE == 0 ? (tid >> 4) : (tid >> 5);
        const int qd = MODE == 0 ? (tid & 15) : (tid & 31);
        const int rstep = MODE == 0 ? kGenWarps * 2 : kGenWarps;
        const uint32_t soff0 =
            MODE == 0 ? rsub * 128 + ((((qd >> 1) ^ (rsub & 7))) << 4) + ((qd & 1) << 3)
                      : (qd >> 4) * 8192 + rsub * 128 + (((((qd & 15) >> 1) ^ (rsub & 7))) << 4) + ((qd & 1) << 3);
        const uint32_t sstep = rstep * 128;
        const bool vec = a.vec_ok != 0;
        const uint32_t w3 = (L.t_w << 20) | sg;
        const bool m_full = MODE == 0 ? (m0 + 128 <= L.N) : (m0 + 128 <= L.K);
        for (int kb = 0; kb < nkb; ++kb) {
            const uint32_t tileA = smem_u32(sA + kb * kAStage) + soff0;
            const bool fullkb = vec && m_full && (MODE == 0 ? (kb * 64 + 64 <= L.K) : (kb * 64 + 64 <= L.N));
            if (fullkb) {
                const int n0 = MODE == 0 ? m0 + rsub : kb * 64 + rsub;
                const int k0 = MODE == 0 ? kb * 64 + 4 * qd : m0 + 4 * qd;
                const int64_t e0 = L.off_w + (int64_t)n0 * L.K + k0;
                const int64_t estep = (int64_t)rstep * L.K;
#pragma unroll 4
                for (int it = 0; it < kItems; ++it) {
                    const uint2 w = gen_w4_fast(L.mu + e0 + it * estep, L.sigma + e0 + it * estep, a.kk.key, a.kk.step,
                                                w3, (uint32_t)(n0 + it * rstep), (uint32_t)(k0 >> 2));
                    sts64(tileA + it * sstep, w);
                }
            } else {
#pragma unroll 1
                for (int it = 0; it < kItems; ++it) {
                    const int n = MODE == 0 ? m0 + rsub + it * rstep : kb * 64 + rsub + it * rstep;
                    const int k = MODE == 0 ? kb * 64 + 4 * qd : m0 + 4 * qd;
                    sts64(tileA + it * sstep, gen_w4(L, a.kk, sg, n, k, vec));
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&wfull[kb]);
        }
        // ------------------------------------------------ epilogue of every row tile
        const int q = warp & 3, h = warp >> 2;
        const int row = 32 * q + lane, m = m0 + row;
        const int nchunks = (a.nb + 15) / 16;
        constexpr int kCStep = kGenWarps / 4;
        const float bias = MODE == 0 ? sbias[row] : 0.0f;
        int tl = 0;
        for (int bt = t0; bt < t1; ++bt, ++tl) {
            const int buf = tl & 1;
            mbar_wait_suspend(&tfull[buf], (tl >> 1) & 1);
            tc_fence_after();
            for (int c = h; c < nchunks; c += kCStep) {
                const int bc0 = bt * NB + c * 16;
                const int nvalid = min(16, a.B - bc0);
                float v[16];
                __syncwarp();
                tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * NB + c * 16, v);
                if (m >= a.M || nvalid <= 0) continue;
                const int64_t base = s * a.out_stride_s + (int64_t)bc0 * a.ldo + m;
                if (a.out_f32) {
                    float* o = reinterpret_cast<float*>(a.out) + base;
                    float rv[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) rv[j] = 0.0f;
                    if (MODE == 0 && a.res_f32) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (j < nvalid) rv[j] = __ldg(a.res_f32 + base + (int64_t)j * a.ldo);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < nvalid) o[(int64_t)j * a.ldo] = v[j] + bias + rv[j];
                } else {
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(a.out) + base;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (j < nvalid) {
                            float z = v[j] + bias;
                            if (MODE == 0 && a.relu) z = fmaxf(z, 0.0f);
                            o[(int64_t)j * a.ldo] = __float2bfloat16_rn(z);
                        }
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
    if (warp == WMMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * NB);
    }
}

// STAGES = 2 (2 CTAs/SM) for the wide layers, whose generation hides the TMA latency; a
// single-M-tile forward layer (the 10-wide output layer: 10 of 128 rows generated) is
// TMA-latency-bound instead and gets 4 stages (prefetch distance 3, 1 CTA/SM).
template <int MODE, int STAGES>
static void launch_gen_gemm_t(dim3 grid, const CUtensorMap& tmB, const TcGenArgs& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(gen_gemm_kernel<MODE, STAGES>), gen::smem_bytes(STAGES));
    gen_gemm_kernel<MODE, STAGES><<<grid, gen::kThreads, gen::smem_bytes(STAGES), st>>>(tmB, a);
}

template <int MODE, int NB>
static void launch_ws(const CUtensorMap& tmB, TcGenArgs a, int S, cudaStream_t st) {
    const int ntb = (a.B + NB - 1) / NB;
    const int mt = (a.M + 127) / 128;
    // one wave: at most kNumSMs CTAs (one per SM); a 149th CTA would run as a second wave
    static const int mode = [] {
        const char* e = std::getenv("BNN_WS_CHUNKS");  // experiment switch: 1 = round the chunk count up
        return e ? std::atoi(e) : 0;
    }();
    const int chunks = std::max(1, std::min(ntb, mode == 1 ? (kNumSMs + mt * S - 1) / (mt * S) : kNumSMs / (mt * S)));
    const int per = (ntb + chunks - 1) / chunks;
    a.nb = NB;
    const dim3 grid(mt, S, (ntb + per - 1) / per);
    ensure_smem_attr(reinterpret_cast<const void*>(gen_gemm_ws_kernel<MODE, NB>), gws::Shape<NB>::kSmem);
    gen_gemm_ws_kernel<MODE, NB><<<grid, gws::kThreads, gws::Shape<NB>::kSmem, st>>>(tmB, a, per);
}

// W-stationary when a sample has several row tiles and no per-row mask / dropout / bias partials
// (the ViT's projections): R ≤ 256 with 256-row tiles (tmB: box 256 rows), R ≤ 768 with 128-row
// tiles (tmB128: box 128 rows; only if given). Returns false if not applicable.
static bool try_ws(const CUtensorMap& tmB, const CUtensorMap* tmB128, const TcGenArgs& a, int S, cudaStream_t st) {
    if (a.mask || a.dbpart || a.drop.on || a.mu_only || (a.B + 255) / 256 < 4) return false;
    if (a.R <= 64 * gws::Shape<256>::kMaxKb) {
        if (a.mode == 0) launch_ws<0, 256>(tmB, a, S, st); else launch_ws<1, 256>(tmB, a, S, st);
        return true;
    }
    if (tmB128 && a.R <= 64 * gws::Shape<128>::kMaxKb) {
        if (a.mode == 0) launch_ws<0, 128>(*tmB128, a, S, st); else launch_ws<1, 128>(*tmB128, a, S, st);
        return true;
    }
    return false;
}

void launch_gen_gemm_ws(const CUtensorMap& tmB256, const CUtensorMap& tmB128, const TcGenArgs& a, int S,
                        cudaStream_t st) {
    if (!try_ws(tmB256, &tmB128, a, S, st)) launch_gen_gemm(tmB256, a, S, st);
}

void launch_gen_gemm(const CUtensorMap& tmB, const TcGenArgs& a, int S, cudaStream_t st) {
    const int ntb = (a.B + 255) / 256;
    if (try_ws(tmB, nullptr, a, S, st)) return;
    dim3 grid((a.M + 127) / 128, S, ntb);
    if (a.mode == 0 && grid.x == 1)
        launch_gen_gemm_t<0, 4>(grid, tmB, a, st);
    else if (a.mode == 0)
        launch_gen_gemm_t<0, 2>(grid, tmB, a, st);
    else
        launch_gen_gemm_t<1, 2>(grid, tmB, a, st);
}

// ============================================================================ K5
namespace wg {
// CTA = 128 n × 112 k weight tile, all S samples; one CTA per SM (TMEM: 2 × 112 columns of
// per-sample dW_s + 112 columns of Σ_s dW_s). 112 = 784 / 7: the C2 layers give 128 full
// tiles + 18 narrow ones = 146 CTAs, one wave on 148 SMs (128-wide tiles left 20 SMs idle;
// 96-wide ones need a second wave). N = 112 MMAs: a tcgen05.mma costs ≈ 130 cycles for any
// N ≤ 256 (profiles/r01/final/mma_bench.txt); two per K = 16 step hide under the ε work.
constexpr int kEpiWarps = 16;
constexpr int kThreads = (kEpiWarps + 2) * 32;  // + TMA warp + MMA warp
constexpr int kStages = 4;
constexpr int kTileK = kWgradTileK;
constexpr int kAStage = 64 * 128 * 2;  // G_sᵀ: 64 b × 128 n (two 64-wide MN blocks)
constexpr int kBStage = 64 * 128 * 2;  // X_s : 64 b × 128 k (two 64-wide MN blocks)
constexpr int kSmem = 1024 + kStages * (kAStage + kBStage) + 256;
}  // namespace wg

__global__ void __launch_bounds__(wg::kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ TcWgradMaps maps, const TcWgradArgs a) {
    using namespace wg;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment as an offset into the __shared__ array: the pointer keeps the shared
    // address space, so plain loads/stores through it compile to LDS/STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // which layer / tile
    int li = 0;
#pragma unroll 1
    while (li + 1 < a.nlayers && (int)blockIdx.x >= a.lay[li + 1].tile_base) ++li;
    const WgradLayer& W = a.lay[li];
    const SampledLayer& L = W.L;
    const int tile = blockIdx.x - W.tile_base;
    const int n0 = (tile / W.ktiles) * 128, k0 = (tile % W.ktiles) * kTileK;
    const CUtensorMap* mapG = &maps.g[li];
    const CUtensorMap* mapX = &maps.x[li];
    const int nbb_all = (a.B + 63) / 64;
    const int nsp = a.nsplit > 1 ? a.nsplit : 1;
    const int per = (nbb_all + nsp - 1) / nsp;
    const int bb0 = blockIdx.y * per;
    const int nbb = max(0, min(nbb_all, bb0 + per) - bb0);  // this split's 64-row blocks
    const int S = a.S;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps);
        }
        mbar_fence_init();
    }
    if (warp == kEpiWarps + 1) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == kEpiWarps) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(mapG);
            tma_prefetch_desc(mapX);
            int it = 0;
            for (int s = 0; s < S; ++s)
                for (int bb = 0; bb < nbb; ++bb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_suspend(&empty[st], ph ^ 1);
                    mbar_arrive_expect_tx(&full[st], kAStage + kBStage);
                    uint8_t* a_st = sA + st * kAStage;
                    const int r0 = 64 * (bb0 + bb);
                    tma_load_3d(mapG, &full[st], a_st, n0, r0, s);
                    tma_load_3d(mapG, &full[st], a_st + 8192, n0 + 64, r0, s);
                    uint8_t* b_st = sB + st * kBStage;
                    tma_load_3d(mapX, &full[st], b_st, k0, r0, W.b_shared ? 0 : s);
                    tma_load_3d(mapX, &full[st], b_st + 8192, k0 + 64, r0, W.b_shared ? 0 : s);
                }
        }
        __syncwarp();
    } else if (warp == kEpiWarps + 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(128, kTileK, 1, 1);
            int it = 0;
            for (int s = 0; s < S; ++s) {
                const int buf = s & 1;
                mbar_wait_suspend(&tempty[buf], ((s >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int bb = 0; bb < nbb; ++bb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait_suspend(&full[st], ph);
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(sA + st * kAStage);
                    const uint32_t bBase = smem_u32(sB + st * kBStage);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t ad = sdesc_sw128(aBase + 2048 * q, 8192, 1024);
                        const uint64_t bd = sdesc_sw128(bBase + 2048 * q, 8192, 1024);
                        // per-sample dW_s (double-buffered) for the ε-weighted acc_ρ ...
                        mma_bf16(tmem + buf * kTileK, ad, bd, idesc, (bb | q) != 0 ? 1u : 0u);
                        // ... and acc_μ = Σ_s dW_s accumulated by the tensor core itself
                        mma_bf16(tmem + 2 * kTileK, ad, bd, idesc, (s | bb | q) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue: ε regeneration + accumulation
        const int q = warp & 3, h = warp >> 2;
        const int n = n0 + 32 * q + lane;
        constexpr int kCW = kTileK / 4;  // columns per epilogue warp (28: four warps per lane quadrant)
        static_assert(kCW == 28, "tmem_ld28 below");
        const int k = k0 + kCW * h;
        const int kend = min(k0 + kTileK, L.K);  // this tile's column range ends here
        const bool kfull = k + kCW <= kend;
        float ar[kCW];
#pragma unroll
        for (int j = 0; j < kCW; ++j) ar[j] = 0.0f;
        for (int s = 0; s < S; ++s) {
            const int buf = s & 1;
            mbar_wait(&tfull[buf], (s >> 1) & 1);
            tc_fence_after();
            float d[kCW];
            __syncwarp();
            tmem_ld28(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kTileK + kCW * h, d);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if (n < L.N && !a.skip_eps && nbb > 0) {
                const uint32_t sgw = ((L.t_w << 20) | (a.kk.s0 + s));
                if (kfull) {
#pragma unroll
                    for (int g = 0; g < kCW / 4; ++g) {
                        const uint4 y = philox10(make_uint4((uint32_t)((k >> 2) + g), (uint32_t)n, sgw,
                                                            a.kk.step), a.kk.key);
                        const float R0 = bm_radius(y.x);
                        const float2 cs0 = bm_sincos(y.y);
                        const float R1 = bm_radius(y.z);
                        const float2 cs1 = bm_sincos(y.w);
                        ar[4 * g + 0] = fmaf(d[4 * g + 0], __fmul_rn(R0, cs0.x), ar[4 * g + 0]);
                        ar[4 * g + 1] = fmaf(d[4 * g + 1], __fmul_rn(R0, cs0.y), ar[4 * g + 1]);
                        ar[4 * g + 2] = fmaf(d[4 * g + 2], __fmul_rn(R1, cs1.x), ar[4 * g + 2]);
                        ar[4 * g + 3] = fmaf(d[4 * g + 3], __fmul_rn(R1, cs1.y), ar[4 * g + 3]);
                    }
                } else {
#pragma unroll
                    for (int g = 0; g < kCW / 4; ++g) {
                        if (k + 4 * g < kend) {
                            const float4 e = eps4(a.kk.key, a.kk.step, a.kk.s0 + s, L.t_w, (uint32_t)n,
                                                  (uint32_t)((k >> 2) + g));
                            float dd[4] = {d[4 * g], d[4 * g + 1], d[4 * g + 2], d[4 * g + 3]};
                            float ee[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) ar[4 * g + j] = fmaf(dd[j], ee[j], ar[4 * g + j]);
                        }
                    }
                }
            }
        }
        // acc_μ from TMEM (complete once the last sample's commit has landed)
        float am[kCW];
        __syncwarp();
        tmem_ld28(tmem + (static_cast<uint32_t>(32 * q) << 16) + 2 * kTileK + kCW * h, am);
        if (S == 0 || nbb == 0) {
#pragma unroll
            for (int j = 0; j < kCW; ++j) am[j] = 0.0f;
        }
        if (nsp > 1 && n < L.N) {  // row split: scaled partials, reduced by launch_wgrad_tc
            const int64_t nk = (int64_t)L.N * L.K, o = (int64_t)n * L.K + k;
            float* pm = a.part + a.part_off[li] + (int64_t)blockIdx.y * 2 * nk + o;
#pragma unroll
            for (int j = 0; j < kCW; ++j) {
                if (k + j < kend) {
                    pm[j] = a.scale * am[j];
                    pm[nk + j] = a.scale * (nbb == 0 ? 0.0f : ar[j]);
                }
            }
        } else if (n < L.N) {
            const int64_t base = L.off_w + (int64_t)n * L.K + k;
            float* pm = a.acc_mu + base;
            float* pr = a.acc_rho + base;
            const bool v4 = ((base & 3) == 0) && kfull;
            if (v4) {
#pragma unroll
                for (int g = 0; g < kCW / 4; ++g) {
                    float4 x = reinterpret_cast<float4*>(pm)[g];
                    float4 y = reinterpret_cast<float4*>(pr)[g];
                    x.x += a.scale * am[4 * g + 0]; x.y += a.scale * am[4 * g + 1];
                    x.z += a.scale * am[4 * g + 2]; x.w += a.scale * am[4 * g + 3];
                    y.x += a.scale * ar[4 * g + 0]; y.y += a.scale * ar[4 * g + 1];
                    y.z += a.scale * ar[4 * g + 2]; y.w += a.scale * ar[4 * g + 3];
                    reinterpret_cast<float4*>(pm)[g] = x;
                    reinterpret_cast<float4*>(pr)[g] = y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < kCW; ++j) {
                    if (k + j < kend) {
                        pm[j] += a.scale * am[j];
                        pr[j] += a.scale * ar[j];
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

void launch_wgrad_tc(const TcWgradMaps& maps, const TcWgradArgs& a, cudaStream_t st) {
    ensure_smem_attr(reinterpret_cast<const void*>(wgrad_tc_kernel), wg::kSmem);
    const WgradLayer& last = a.lay[a.nlayers - 1];
    const int ntiles = last.tile_base + last.mtiles * last.ktiles;
    const int nsp = a.nsplit > 1 ? a.nsplit : 1;
    wgrad_tc_kernel<<<dim3(ntiles, nsp), wg::kThreads, wg::kSmem, st>>>(maps, a);
    if (nsp > 1)
        for (int l = 0; l < a.nlayers; ++l)
            launch_wgrad_split_reduce(a.part + a.part_off[l], nsp, (int64_t)a.lay[l].L.N * a.lay[l].L.K,
                                      a.lay[l].L.off_w, a.acc_mu, a.acc_rho, st);
}

}  // namespace bnn
