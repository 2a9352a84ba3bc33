// kernels_simt.cu — HBM-bound elementwise/reduction kernels (K1, K6, K7, K8, K10) and the
// FP32 SIMT sampled-GEMM kernels of the FP32 parity mode (K11).
//
// Equations (DESIGN.md §1 cites each to PAPER.md):
//   σ = softplus(ρ)                                          K7, R1
//   W_s[n][k] = fma(σ, ε_s, μ) rounded once in fp32           PAPER.md:159 (Alg. 1 l.6)
//   CE: ℓ = logsumexp(z) − z_y, dℓ/dz = softmax(z) − onehot    PAPER.md:162, R5/R6
//   MSE: ℓ = Σ_o (z−y)², dℓ/dz = 2(z−y)                        PAPER.md:162, :320, R7
//   grad_μ = acc_μ + μ/|D|; grad_ρ = sigmoid(ρ)(acc_ρ + (σ − 1/σ)/|D|)
//   KL = ½ Σ (σ² + μ² − 1 − 2 ln σ)
#include <algorithm>

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace bnn {

void ensure_smem_attr(const void* func, int bytes) {
    static std::mutex m;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(m);
    if (done.insert({func, dev}).second)
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}


// ====================================================================== K7: σ prologue
__global__ void sigma_kernel(const float* __restrict__ rho, float* __restrict__ sigma,
                             int64_t n) {
    const int64_t n4 = n / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 r = reinterpret_cast<const float4*>(rho)[i];
        reinterpret_cast<float4*>(sigma)[i] =
            make_float4(softplus_f(r.x), softplus_f(r.y), softplus_f(r.z), softplus_f(r.w));
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        sigma[i] = softplus_f(rho[i]);
}

void launch_sigma(const float* rho, float* sigma, int64_t n, cudaStream_t st) {
    int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, kNumSMs * 8);
    sigma_kernel<<<grid, 256, 0, st>>>(rho, sigma, n);
}

// ====================================================================== K8: finalize + KL
__device__ __forceinline__ double fin_one(float mu, float rho, float am, float ar, float invD,
                                          float& gm, float& gr) {
    const float sg = softplus_f(rho);
    gm = am + mu * invD;
    gr = sigmoid_f(rho) * (ar + (sg - 1.0f / sg) * invD);
    const float ls = log_sigma_f(rho, sg);
    return 0.5 * ((double)sg * sg + (double)mu * mu - 1.0 - 2.0 * (double)ls);
}

__global__ void __launch_bounds__(256) finalize_kernel(
    const float* __restrict__ mu, const float* __restrict__ rho, const float* __restrict__ acc_mu,
    const float* __restrict__ acc_rho, int64_t P, float invD, float* __restrict__ grad_mu,
    float* __restrict__ grad_rho, double* __restrict__ kl_partials, int mcd) {
    double kl = 0.0;
    if (mcd) {  // MC dropout (R25): grad_μ = the data gradient, no ρ, no prior term
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
            grad_mu[i] = acc_mu[i];
            grad_rho[i] = 0.0f;
        }
        if (threadIdx.x == 0) kl_partials[blockIdx.x] = 0.0;
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t P4 = P / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P4; i += stride) {
        const float4 m = reinterpret_cast<const float4*>(mu)[i];
        const float4 r = reinterpret_cast<const float4*>(rho)[i];
        const float4 a = reinterpret_cast<const float4*>(acc_mu)[i];
        const float4 b = reinterpret_cast<const float4*>(acc_rho)[i];
        float4 gm, gr;
        kl += fin_one(m.x, r.x, a.x, b.x, invD, gm.x, gr.x);
        kl += fin_one(m.y, r.y, a.y, b.y, invD, gm.y, gr.y);
        kl += fin_one(m.z, r.z, a.z, b.z, invD, gm.z, gr.z);
        kl += fin_one(m.w, r.w, a.w, b.w, invD, gm.w, gr.w);
        reinterpret_cast<float4*>(grad_mu)[i] = gm;
        reinterpret_cast<float4*>(grad_rho)[i] = gr;
    }
    for (int64_t i = 4 * P4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
        float gm, gr;
        kl += fin_one(mu[i], rho[i], acc_mu[i], acc_rho[i], invD, gm, gr);
        grad_mu[i] = gm;
        grad_rho[i] = gr;
    }
    __shared__ double red[8];
    kl = warp_sum(kl);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = kl;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        kl_partials[blockIdx.x] = t;
    }
}

__global__ void finalize_loss_kernel(const double* __restrict__ kl_partials, int n,
                                     const float* __restrict__ Ldata, double invD,
                                     float* __restrict__ loss) {
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += kl_partials[i];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double kl = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) kl += red[w];
        loss[0] = (float)((double)Ldata[0] + kl * invD);
        loss[1] = (float)kl;
    }
}

int finalize_partials_count(int64_t P) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((P / 4 + 255) / 256, kNumSMs * 8));
}

void launch_finalize(int mcd, const float* mu, const float* rho, const float* acc_mu,
                      const float* acc_rho, const float* Ldata, int64_t P, double D,
                      float* grad_mu, float* grad_rho, double* kl_partials, int n_part,
                      float* loss, cudaStream_t st) {
    finalize_kernel<<<n_part, 256, 0, st>>>(mu, rho, acc_mu, acc_rho, P, (float)(1.0 / D),
                                            grad_mu, grad_rho, kl_partials, mcd);
    finalize_loss_kernel<<<1, 1024, 0, st>>>(kl_partials, n_part, Ldata, 1.0 / D, loss);
}

// ---------------------------------------------------------------- K8 + Adam
// The finalize of K8 followed, in the same pass over the parameters, by the Adam update the
// paper's Alg. 1 l.13 / Alg. 2 l.16 name (Kingma & Ba Alg. 1):
//   m ← β1 m + (1−β1) g;  v ← β2 v + (1−β2) g²;  θ ← θ − lr·(m/bc1)/(√(v/bc2) + ε)
// for θ ∈ {μ, ρ}. KL and the loss use the parameters before the update. One HBM pass:
// reads μ, ρ, acc_μ, acc_ρ and the four moments, writes μ, ρ and the moments (+ the gradients
// when requested): 56 B/param (64 with gradients).
__device__ __forceinline__ void adam_one(float& th, float g, float& m, float& v, const AdamHyper& h) {
    m = __fmaf_rn(h.beta1, m, h.omb1 * g);
    v = __fmaf_rn(h.beta2, v, h.omb2 * (g * g));
    const float mhat = m / h.bc1;
    const float vhat = v / h.bc2;
    th = th - h.lr * mhat / (sqrtf(vhat) + h.eps);
}

__global__ void __launch_bounds__(256) finalize_adam_kernel(
    float* __restrict__ mu, float* __restrict__ rho, const float* __restrict__ acc_mu,
    const float* __restrict__ acc_rho, int64_t P, float invD, const AdamHyper h,
    float* __restrict__ m_mu, float* __restrict__ v_mu, float* __restrict__ m_rho,
    float* __restrict__ v_rho, float* __restrict__ grad_mu, float* __restrict__ grad_rho,
    double* __restrict__ kl_partials) {
    double kl = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t P4 = P / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P4; i += stride) {
        float4 m = reinterpret_cast<const float4*>(mu)[i];
        float4 r = reinterpret_cast<const float4*>(rho)[i];
        const float4 a = reinterpret_cast<const float4*>(acc_mu)[i];
        const float4 b = reinterpret_cast<const float4*>(acc_rho)[i];
        float4 mm = reinterpret_cast<const float4*>(m_mu)[i];
        float4 vm = reinterpret_cast<const float4*>(v_mu)[i];
        float4 mr = reinterpret_cast<const float4*>(m_rho)[i];
        float4 vr = reinterpret_cast<const float4*>(v_rho)[i];
        float4 gm, gr;
        kl += fin_one(m.x, r.x, a.x, b.x, invD, gm.x, gr.x);
        kl += fin_one(m.y, r.y, a.y, b.y, invD, gm.y, gr.y);
        kl += fin_one(m.z, r.z, a.z, b.z, invD, gm.z, gr.z);
        kl += fin_one(m.w, r.w, a.w, b.w, invD, gm.w, gr.w);
        adam_one(m.x, gm.x, mm.x, vm.x, h); adam_one(r.x, gr.x, mr.x, vr.x, h);
        adam_one(m.y, gm.y, mm.y, vm.y, h); adam_one(r.y, gr.y, mr.y, vr.y, h);
        adam_one(m.z, gm.z, mm.z, vm.z, h); adam_one(r.z, gr.z, mr.z, vr.z, h);
        adam_one(m.w, gm.w, mm.w, vm.w, h); adam_one(r.w, gr.w, mr.w, vr.w, h);
        reinterpret_cast<float4*>(mu)[i] = m;
        reinterpret_cast<float4*>(rho)[i] = r;
        reinterpret_cast<float4*>(m_mu)[i] = mm;
        reinterpret_cast<float4*>(v_mu)[i] = vm;
        reinterpret_cast<float4*>(m_rho)[i] = mr;
        reinterpret_cast<float4*>(v_rho)[i] = vr;
        if (grad_mu) reinterpret_cast<float4*>(grad_mu)[i] = gm;
        if (grad_rho) reinterpret_cast<float4*>(grad_rho)[i] = gr;
    }
    for (int64_t i = 4 * P4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
        float gm, gr;
        kl += fin_one(mu[i], rho[i], acc_mu[i], acc_rho[i], invD, gm, gr);
        adam_one(mu[i], gm, m_mu[i], v_mu[i], h);
        adam_one(rho[i], gr, m_rho[i], v_rho[i], h);
        if (grad_mu) grad_mu[i] = gm;
        if (grad_rho) grad_rho[i] = gr;
    }
    __shared__ double red[8];
    kl = warp_sum(kl);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = kl;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        kl_partials[blockIdx.x] = t;
    }
}

void launch_finalize_adam(float* mu, float* rho, const float* acc_mu, const float* acc_rho,
                          const float* Ldata, int64_t P, double D, const AdamHyper& h,
                          float* m_mu, float* v_mu, float* m_rho, float* v_rho, float* grad_mu,
                          float* grad_rho, double* kl_partials, int n_part, float* loss,
                          cudaStream_t st) {
    finalize_adam_kernel<<<n_part, 256, 0, st>>>(mu, rho, acc_mu, acc_rho, P, (float)(1.0 / D), h,
                                                 m_mu, v_mu, m_rho, v_rho, grad_mu, grad_rho,
                                                 kl_partials);
    finalize_loss_kernel<<<1, 1024, 0, st>>>(kl_partials, n_part, Ldata, 1.0 / D, loss);
}

// ====================================================================== K6: loss head
__global__ void loss_head_kernel(const float* __restrict__ logits, int rows, int B, int O,
                                 int loss_kind, const int32_t* __restrict__ ycls,
                                 const float* __restrict__ yreg, void* __restrict__ dz, int ldg,
                                 int dz_bf16, float* __restrict__ lossrow,
                                 float* __restrict__ dz_f32) {
    const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const int b = warp % B;
    const float* z = logits + (int64_t)warp * O;
    float loss = 0.0f;
    auto put = [&](int k, float v) {
        if (dz_f32 && k < O) dz_f32[(int64_t)warp * O + k] = v;
        if (dz_bf16)
            reinterpret_cast<__nv_bfloat16*>(dz)[(int64_t)warp * ldg + k] = __float2bfloat16_rn(v);
        else
            reinterpret_cast<float*>(dz)[(int64_t)warp * ldg + k] = v;
    };
    if (loss_kind == 0) {  // CE
        float m = -INFINITY;
        for (int k = lane; k < O; k += 32) m = fmaxf(m, z[k]);
        m = warp_max(m);
        float se = 0.0f;
        for (int k = lane; k < O; k += 32) se += expf(z[k] - m);
        se = warp_sum(se);
        const float lse = m + logf(se);
        // a label outside [0, O) is a caller error: no out-of-bounds read, a NaN loss (the
        // loss read returns BNN_ERR_NUMERIC) and a zero gradient seed for the example
        const int y0 = ycls[b];
        const bool ok = y0 >= 0 && y0 < O;
        const int y = ok ? y0 : 0;
        for (int k = lane; k < O; k += 32) put(k, ok ? expf(z[k] - lse) - (k == y ? 1.0f : 0.0f) : 0.0f);
        loss = ok ? lse - z[y] : __int_as_float(0x7fc00000);
    } else {  // MSE
        float l = 0.0f;
        for (int k = lane; k < O; k += 32) {
            const float d = z[k] - yreg[(int64_t)b * O + k];
            l += d * d;
            put(k, 2.0f * d);
        }
        loss = warp_sum(l);
    }
    for (int k = O + lane; k < ldg; k += 32) put(k, 0.0f);
    if (lane == 0) lossrow[warp] = loss;
}

void launch_loss_head(const float* logits, int S, int B, int O, int loss_kind,
                      const int32_t* ycls, const float* yreg, void* dz, int ldg, bool dz_bf16,
                      float* lossrow, float* dz_f32, cudaStream_t st) {
    const int rows = S * B;
    loss_head_kernel<<<(rows + 7) / 8, 256, 0, st>>>(logits, rows, B, O, loss_kind, ycls, yreg,
                                                     dz, ldg, dz_bf16 ? 1 : 0, lossrow, dz_f32);
}

__global__ void loss_reduce_kernel(const float* __restrict__ lossrow, int n, float scale,
                                   float* __restrict__ acc_slot) {
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += (double)lossrow[i];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        acc_slot[0] = (float)((double)acc_slot[0] + s * (double)scale);
    }
}

void launch_loss_reduce(const float* lossrow, int n, float scale, float* acc_slot,
                        cudaStream_t st) {
    loss_reduce_kernel<<<1, 1024, 0, st>>>(lossrow, n, scale, acc_slot);
}

// ---------------------------------------------------------------- exact aggregation
// Loss of the mean prediction over all S samples: CE of the arithmetic
// mean of the true-class probabilities, or MSE of the mean output. The per-rank statistic is
// a plain fp32 sum over this rank's samples (CE: Σ_s p_{s,b,y}, width 1; MSE: Σ_s ŷ_{s,b,o},
// width O), accumulated sample by sample in order (deterministic), merged over the sample
// groups, then turned into per-sample gradient seeds.
__global__ void mean_stats_kernel(const float* __restrict__ logits, int Sc, int B, int O,
                                  int loss_kind, const int32_t* __restrict__ ycls,
                                  float* __restrict__ stats, int n_prev) {
    if (loss_kind == 2) {  // Gaussian NLL: Welford (mean, M2) per (example, output), samples in order
        const int i = blockIdx.x * blockDim.x + threadIdx.x;
        if (i >= B * O) return;
        const int b = i / O, o = i - b * O;
        float* pm = stats + (int64_t)b * 2 * O + o;
        float mean = pm[0], m2 = pm[O];
        for (int s = 0; s < Sc; ++s) {
            const float x = logits[(int64_t)s * B * O + i];
            const float d = x - mean;
            mean += d / (float)(n_prev + s + 1);
            m2 = fmaf(d, x - mean, m2);
        }
        pm[0] = mean;
        pm[O] = m2;
        return;
    }
    if (loss_kind == 0) {  // CE: one warp per example, lanes over samples, fixed-order warp sum
        const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        const int lane = threadIdx.x & 31;
        if (b >= B) return;
        const int y0 = ycls[b];
        const int y = (y0 >= 0 && y0 < O) ? y0 : 0;  // out-of-range label: NaN statistic below
        float part = (y0 >= 0 && y0 < O) ? 0.0f : __int_as_float(0x7fc00000);
        for (int s = lane; s < Sc; s += 32) {
            const float* z = logits + ((int64_t)s * B + b) * O;
            float m = z[0];
            for (int k = 1; k < O; ++k) m = fmaxf(m, z[k]);
            float se = 0.0f;
            for (int k = 0; k < O; ++k) se += expf(z[k] - m);
            part += expf(z[y] - m) / se;
        }
        part = warp_sum(part);
        if (lane == 0) stats[b] += part;
    } else {  // MSE: one thread per (example, output), samples in order
        const int i = blockIdx.x * blockDim.x + threadIdx.x;
        if (i >= B * O) return;
        float acc = stats[i];
        for (int s = 0; s < Sc; ++s) acc += logits[(int64_t)s * B * O + i];
        stats[i] = acc;
    }
}

void launch_mean_stats(const float* logits, int Sc, int B, int O, int loss_kind,
                       const int32_t* ycls, float* stats, int n_prev, cudaStream_t st) {
    if (loss_kind == 0)
        mean_stats_kernel<<<(B + 7) / 8, 256, 0, st>>>(logits, Sc, B, O, loss_kind, ycls, stats, n_prev);
    else
        mean_stats_kernel<<<(B * O + 127) / 128, 128, 0, st>>>(logits, Sc, B, O, loss_kind, ycls, stats,
                                                               n_prev);
}

// CE / MSE: out[i] = Σ over ranks r with r % G == g (the sample groups of data group g), in
// rank order. Gaussian NLL (gnll_O > 0): per (example, output) the (mean, M2) of every such rank
// (n_rank samples each) merged in rank order by Chan et al.'s pairwise update.
__global__ void mean_merge_kernel(const float* __restrict__ gathered, int world, int G, int g,
                                  int64_t n, float* __restrict__ out, int gnll_O, int n_rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gnll_O > 0) {
        if (i >= n / 2) return;
        const int64_t b = i / gnll_O, o = i - b * gnll_O;
        const int64_t im = b * 2 * gnll_O + o, iv = im + gnll_O;
        float mean = 0.0f, m2 = 0.0f, na = 0.0f;
        for (int r = g; r < world; r += G) {
            const float mr = gathered[(int64_t)r * n + im], vr = gathered[(int64_t)r * n + iv];
            const float nb = (float)n_rank, nn = na + nb;
            const float d = mr - mean;
            mean = fmaf(d, nb / nn, mean);
            m2 = m2 + vr + d * d * (na * nb / nn);
            na = nn;
        }
        out[im] = mean;
        out[iv] = m2;
        return;
    }
    if (i >= n) return;
    float acc = 0.0f;
    for (int r = g; r < world; r += G) acc += gathered[(int64_t)r * n + i];
    out[i] = acc;
}

void launch_mean_merge(const float* gathered, int world, int G, int g, int64_t n, float* out,
                       int gnll_O, int n_rank, cudaStream_t st) {
    mean_merge_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(gathered, world, G, g, n, out, gnll_O, n_rank);
}

// Gradient seed of the mean-prediction loss for each (s, b) row, unscaled like loss_head_kernel
// (the 1/(S·B) or 1/(S·B·O) scale is applied downstream):
//   CE:  dz_k = (S·p_{s,y}/Σ_s' p_{s',y}) · (p_k − [k = y])      (= (p_y/P̄)(p − onehot))
//   MSE: dz_o = 2·(Σ_s' ŷ_{s',o}/S − y_o)
__global__ void mean_loss_head_kernel(const float* __restrict__ logits, int rows, int B, int O,
                                      int loss_kind, const int32_t* __restrict__ ycls,
                                      const float* __restrict__ yreg,
                                      const float* __restrict__ gstats, float S_glob,
                                      void* __restrict__ dz, int ldg, int dz_bf16,
                                      float* __restrict__ dz_f32) {
    const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const int b = warp % B;
    const float* z = logits + (int64_t)warp * O;
    auto put = [&](int k, float v) {
        if (dz_f32 && k < O) dz_f32[(int64_t)warp * O + k] = v;
        if (dz_bf16)
            reinterpret_cast<__nv_bfloat16*>(dz)[(int64_t)warp * ldg + k] = __float2bfloat16_rn(v);
        else
            reinterpret_cast<float*>(dz)[(int64_t)warp * ldg + k] = v;
    };
    if (loss_kind == 0) {
        float m = -INFINITY;
        for (int k = lane; k < O; k += 32) m = fmaxf(m, z[k]);
        m = warp_max(m);
        float se = 0.0f;
        for (int k = lane; k < O; k += 32) se += expf(z[k] - m);
        se = warp_sum(se);
        const float lse = m + logf(se);
        const int y0 = ycls[b];
        const int y = (y0 >= 0 && y0 < O) ? y0 : 0;  // out-of-range label: the statistic is NaN already
        const float w = S_glob * expf(z[y] - lse) / gstats[b];
        for (int k = lane; k < O; k += 32) put(k, w * (expf(z[k] - lse) - (k == y ? 1.0f : 0.0f)));
    } else if (loss_kind == 2) {
        // Gaussian NLL of the predictive: m, v = M2/S + 1e-6 (reading R24);
        // seed (unscaled): (ŷ − m)/v − (y − m)/v − (y − m)²(ŷ − m)/v²
        for (int k = lane; k < O; k += 32) {
            const float m = gstats[(int64_t)b * 2 * O + k];
            const float v = gstats[(int64_t)b * 2 * O + O + k] / S_glob + 1e-6f;
            const float e = z[k] - m, d = yreg[(int64_t)b * O + k] - m;
            put(k, (e - d) / v - d * d * e / (v * v));
        }
    } else {
        for (int k = lane; k < O; k += 32)
            put(k, 2.0f * (gstats[(int64_t)b * O + k] / S_glob - yreg[(int64_t)b * O + k]));
    }
    for (int k = O + lane; k < ldg; k += 32) put(k, 0.0f);
}

void launch_mean_loss_head(const float* logits, int S, int B, int O, int loss_kind,
                           const int32_t* ycls, const float* yreg, const float* gstats,
                           int S_glob, void* dz, int ldg, bool dz_bf16, float* dz_f32,
                           cudaStream_t st) {
    const int rows = S * B;
    mean_loss_head_kernel<<<(rows + 7) / 8, 256, 0, st>>>(logits, rows, B, O, loss_kind, ycls, yreg,
                                                          gstats, (float)S_glob, dz, ldg,
                                                          dz_bf16 ? 1 : 0, dz_f32);
}

// acc_slot += scale · Σ_b ℓ_b with ℓ_b = −ln(Σ_s p_y / S) (CE) or Σ_o (Σ_s ŷ_o / S − y_o)² (MSE)
__global__ void mean_loss_value_kernel(const float* __restrict__ gstats, int B, int O,
                                       int loss_kind, const float* __restrict__ yreg,
                                       float S_glob, float scale, float* __restrict__ acc_slot) {
    __shared__ double red[32];
    double t = 0.0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        if (loss_kind == 0) {
            t += -log((double)gstats[b] / (double)S_glob);
        } else if (loss_kind == 2) {
            for (int k = 0; k < O; ++k) {
                const double m = gstats[(int64_t)b * 2 * O + k];
                const double v = (double)gstats[(int64_t)b * 2 * O + O + k] / (double)S_glob + 1e-6;
                const double d = (double)yreg[(int64_t)b * O + k] - m;
                t += 0.5 * log(6.283185307179586 * v) + d * d / (2.0 * v);
            }
        } else {
            for (int k = 0; k < O; ++k) {
                const double d = (double)gstats[(int64_t)b * O + k] / (double)S_glob -
                                 (double)yreg[(int64_t)b * O + k];
                t += d * d;
            }
        }
    }
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        acc_slot[0] = (float)((double)acc_slot[0] + s * (double)scale);
    }
}

void launch_mean_loss_value(const float* gstats, int B, int O, int loss_kind, const float* yreg,
                            int S_glob, float scale, float* acc_slot, cudaStream_t st) {
    mean_loss_value_kernel<<<1, 1024, 0, st>>>(gstats, B, O, loss_kind, yreg, (float)S_glob, scale,
                                               acc_slot);
}

// ====================================================================== K1: ε fill / bench
__global__ void eps_fill_kernel(EpsKey key, uint32_t step, uint32_t s, uint32_t t, uint32_t r0,
                                uint32_t nr, uint32_t c0, uint32_t nc, float* __restrict__ out) {
    const uint64_t n = (uint64_t)nr * nc;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(i / nc), c = (uint32_t)(i % nc);
        out[i] = eps1(key, step, s, t, r0 + r, c0 + c);
    }
}

void launch_eps_fill(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r0,
                     uint32_t nr, uint32_t c0, uint32_t nc, float* out, cudaStream_t st) {
    const uint64_t n = (uint64_t)nr * nc;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)kNumSMs * 16);
    eps_fill_kernel<<<std::max(grid, 1), 256, 0, st>>>(make_key(seed), step, s, t, r0, nr, c0,
                                                       nc, out);
}

__global__ void __launch_bounds__(256) eps_bench_kernel(uint64_t n4, EpsKey key,
                                                        float* __restrict__ sink) {
    float acc = 0.0f;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 e = eps4(key, 0u, 0u, 0u, (uint32_t)(i >> 32), (uint32_t)i);
        acc += (e.x + e.y) + (e.z + e.w);
    }
    acc = warp_sum(acc);
    __shared__ float red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.0f;
        for (int w = 0; w < 8; ++w) t += red[w];
        sink[blockIdx.x] = t;
    }
}

void launch_eps_bench(uint64_t n4, uint64_t seed, float* sink, int grid, cudaStream_t st) {
    eps_bench_kernel<<<grid, 256, 0, st>>>(n4, make_key(seed), sink);
}

// every EPS-v1 transform input: which 0 → R(k) for k = 1..2^24 (u = k·2^-24),
// which 1/2 → cos/sin(2π v/2^24) for v = 0..2^24-1
__global__ void eps_table_kernel(int which, float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (1u << 24)) return;
    if (which == 0) {
        out[i] = bm_radius(i << 8);  // (a >> 8) + 1 = i + 1
    } else {
        const float2 cs = bm_sincos(i << 8);
        out[i] = which == 1 ? cs.x : cs.y;
    }
}

void launch_eps_table(int which, float* out, cudaStream_t st) {
    eps_table_kernel<<<(1 << 24) / 256, 256, 0, st>>>(which, out);
}

// ====================================================================== K10: predict stats
__global__ void predict_stats_kernel(const float* __restrict__ logits, int S, int B, int O,
                                     int loss_kind, float* __restrict__ mean,
                                     float* __restrict__ m2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (b, o)
    if (i >= B * O) return;
    const int b = i / O, o = i % O;
    auto prob = [&](int s) -> float {
        const float* z = logits + ((int64_t)s * B + b) * O;
        if (loss_kind != 0) return z[o];
        float m = z[0];
        for (int k = 1; k < O; ++k) m = fmaxf(m, z[k]);
        float se = 0.0f;
        for (int k = 0; k < O; ++k) se += expf(z[k] - m);
        return expf(z[o] - m) / se;
    };
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += prob(s);
    const double mu = acc / S;
    double v = 0.0;
    for (int s = 0; s < S; ++s) {
        const double d = prob(s) - mu;
        v += d * d;
    }
    mean[i] = (float)mu;
    m2[i] = (float)v;
}

void launch_predict_stats(const float* logits, int S, int B, int O, int loss_kind, float* mean,
                          float* m2, cudaStream_t st) {
    predict_stats_kernel<<<(B * O + 255) / 256, 256, 0, st>>>(logits, S, B, O, loss_kind, mean,
                                                              m2);
}

__global__ void predict_merge_kernel(const float* __restrict__ means, const float* __restrict__ m2s,
                                     const float* __restrict__ counts, int R, int BO,
                                     float* __restrict__ mean, float* __restrict__ var) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= BO) return;
    double n = 0.0, mu = 0.0, M2 = 0.0;
    for (int r = 0; r < R; ++r) {  // Chan et al. pairwise update, fixed rank order
        const double nr = counts[r];
        const double mr = means[(int64_t)r * BO + i];
        const double n_new = n + nr;
        const double d = mr - mu;
        mu += d * nr / n_new;
        M2 += (double)m2s[(int64_t)r * BO + i] + d * d * n * nr / n_new;
        n = n_new;
    }
    mean[i] = (float)mu;
    var[i] = (float)(M2 / n);
}

void launch_predict_merge(const float* means, const float* m2s, const float* counts, int R,
                          int BO, float* mean, float* var, cudaStream_t st) {
    predict_merge_kernel<<<(BO + 255) / 256, 256, 0, st>>>(means, m2s, counts, R, BO, mean, var);
}

// ====================================================================== input cast
__global__ void to_bf16_kernel(const float* __restrict__ x, int B, int K, int ldx,
                               __nv_bfloat16* __restrict__ out) {
    const int64_t n = (int64_t)B * ldx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(i / ldx), k = (int)(i % ldx);
        out[i] = __float2bfloat16_rn(k < K ? x[(int64_t)b * K + k] : 0.0f);
    }
}

void launch_to_bf16(const float* x, int B, int K, int ldx, void* out, cudaStream_t st) {
    const int64_t n = (int64_t)B * ldx;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
    to_bf16_kernel<<<grid, 256, 0, st>>>(x, B, K, ldx, reinterpret_cast<__nv_bfloat16*>(out));
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, int64_t n, float* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __bfloat162float(x[i]);
}
void launch_bf16_to_f32(const void* x, int64_t n, float* y, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
    bf16_to_f32_kernel<<<std::max(grid, 1), 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), n, y);
}

// ====================================================================== K11: FP32 SIMT GEMMs
constexpr int TB = 64, TK = 16;

__global__ void __launch_bounds__(256) fwd_fp32_kernel(SampledLayer L, SampleKeys kk, DropArgs d, int B,
                                                       const float* __restrict__ A,
                                                       int64_t strideA, float* __restrict__ Z,
                                                       int64_t strideZ, int relu) {
    __shared__ float As[TK][TB + 4];  // [k][b]
    __shared__ float Ws[TK][TB + 4];  // [k][n]
    __shared__ float bias[TB];
    const int n0 = blockIdx.x * TB, b0 = blockIdx.y * TB, s = blockIdx.z;
    const uint32_t sg = kk.s0 + s;
    const float* Ag = A + s * strideA;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = L.N, K = L.K;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        {
            const int bb = tid >> 2, kq = (tid & 3) * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = k0 + kq + j;
                As[kq + j][bb] = (b0 + bb < B && k < K) ? Ag[(int64_t)(b0 + bb) * K + k] : 0.0f;
            }
        }
        {
            const int nn = tid >> 2, kq = tid & 3, n = n0 + nn, kb = k0 + 4 * kq;
            float w[4] = {0.f, 0.f, 0.f, 0.f};
            if (n < N && kb < K) {
                const float4 e = eps4(kk.key, kk.step, sg, L.t_w, n, kb >> 2);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (kb + j < K) {
                        const int64_t i = L.off_w + (int64_t)n * K + kb + j;
                        w[j] = __fmaf_rn(L.sigma[i], eps_get(e, j), L.mu[i]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) Ws[4 * kq + j][nn] = w[j];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TK; ++q) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[q][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = Ws[q][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (tid < TB) {
        const int n = n0 + tid;
        bias[tid] = n < N ? __fmaf_rn(L.sigma[L.off_b + n], eps1(kk.key, kk.step, sg, L.t_b, 0, n),
                                      L.mu[L.off_b + n])
                          : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b = b0 + ty * 4 + i;
        if (b >= B) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= N) continue;
            float v = acc[i][j] + bias[tx * 4 + j];
            if (relu) v = fmaxf(v, 0.0f);
            if (d.on)
                v = dropout_keep(kk.key, kk.step, sg, (uint32_t)d.layer, (uint32_t)(d.b_off + b), (uint32_t)n, d.p24)
                        ? v * d.inv_keep : 0.0f;
            Z[s * strideZ + (int64_t)b * N + n] = v;
        }
    }
}

void launch_fwd_fp32(const SampledLayer& L, const SampleKeys& k, const DropArgs& d, int S, int B, const float* A,
                     int64_t strideA, float* Z, int64_t strideZ, bool relu, cudaStream_t st) {
    dim3 grid((L.N + TB - 1) / TB, (B + TB - 1) / TB, S);
    fwd_fp32_kernel<<<grid, 256, 0, st>>>(L, k, d, B, A, strideA, Z, strideZ, relu ? 1 : 0);
}

__global__ void __launch_bounds__(256) dgrad_fp32_kernel(SampledLayer L, SampleKeys kk, DropArgs d, int B,
                                                         const float* __restrict__ G,
                                                         int64_t strideG,
                                                         const float* __restrict__ Ap,
                                                         int64_t strideA, float* __restrict__ dA,
                                                         int64_t strideD) {
    __shared__ float Gs[TK][TB + 4];  // [n][b]
    __shared__ float Ws[TK][TB + 4];  // [n][k]
    const int kt0 = blockIdx.x * TB, b0 = blockIdx.y * TB, s = blockIdx.z;
    const uint32_t sg = kk.s0 + s;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = L.N, K = L.K;
    const float* Gg = G + s * strideG;
    float acc[4][4] = {};
    for (int n0 = 0; n0 < N; n0 += TK) {
        {
            const int bb = tid >> 2, nq = (tid & 3) * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + nq + j;
                Gs[nq + j][bb] = (b0 + bb < B && n < N) ? Gg[(int64_t)(b0 + bb) * N + n] : 0.0f;
            }
        }
        {
            const int nn = tid >> 4, kq = tid & 15, n = n0 + nn, kb = kt0 + 4 * kq;
            float w[4] = {0.f, 0.f, 0.f, 0.f};
            if (n < N && kb < K) {
                const float4 e = eps4(kk.key, kk.step, sg, L.t_w, n, kb >> 2);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (kb + j < K) {
                        const int64_t i = L.off_w + (int64_t)n * K + kb + j;
                        w[j] = __fmaf_rn(L.sigma[i], eps_get(e, j), L.mu[i]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) Ws[nn][4 * kq + j] = w[j];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TK; ++q) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = Gs[q][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = Ws[q][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b = b0 + ty * 4 + i;
        if (b >= B) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = kt0 + tx * 4 + j;
            if (k >= K) continue;
            // ReLU (and, under MC dropout, the keep mask: the stored input is 0 where dropped)
            // (Ap == null: no activation mask — the ViT's projections, whose nonlinearities are
            // separate kernels)
            const float m = Ap == nullptr ? 1.0f
                            : Ap[s * strideA + (int64_t)b * K + k] > 0.0f ? (d.on ? d.inv_keep : 1.0f) : 0.0f;
            dA[s * strideD + (int64_t)b * K + k] = acc[i][j] * m;
        }
    }
}

void launch_dgrad_fp32(const SampledLayer& L, const SampleKeys& k, const DropArgs& d, int S, int B, const float* G,
                       int64_t strideG, const float* Aprev, int64_t strideA, float* dA,
                       int64_t strideD, cudaStream_t st) {
    dim3 grid((L.K + TB - 1) / TB, (B + TB - 1) / TB, S);
    dgrad_fp32_kernel<<<grid, 256, 0, st>>>(L, k, d, B, G, strideG, Aprev, strideA, dA, strideD);
}

__global__ void __launch_bounds__(256) wgrad_fp32_kernel(SampledLayer L, SampleKeys kk, int S,
                                                         int B, const float* __restrict__ G,
                                                         int64_t strideG,
                                                         const float* __restrict__ A,
                                                         int64_t strideA, float scale,
                                                         float* __restrict__ acc_mu,
                                                         float* __restrict__ acc_rho, int rows_per,
                                                         float* __restrict__ part) {
    __shared__ float Gs[TK][TB + 4];  // [b][n]
    __shared__ float As[TK][TB + 4];  // [b][k]
    const int kt0 = blockIdx.x * TB, n0 = blockIdx.y * TB;
    // row split z (the ViT's token rows): rows [z·rows_per, …) of every sample; the scaled
    // partial sums go to part[z][μ|ρ][N·K] and a fixed-order reduction adds them to acc
    const int r0 = blockIdx.z * rows_per, r1 = min(B, r0 + rows_per);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = L.N, K = L.K;
    float am[4][4] = {}, ar[4][4] = {};
    for (int s = 0; s < S; ++s) {
        const float* Gg = G + s * strideG;
        const float* Ag = A + s * strideA;
        float d[4][4] = {};
        for (int b0 = r0; b0 < r1; b0 += TK) {
            {
                const int bb = tid >> 4, q = (tid & 15) * 4;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int n = n0 + q + j, k = kt0 + q + j, b = b0 + bb;
                    Gs[bb][q + j] = (b < r1 && n < N) ? Gg[(int64_t)b * N + n] : 0.0f;
                    As[bb][q + j] = (b < r1 && k < K) ? Ag[(int64_t)b * K + k] : 0.0f;
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < TK; ++q) {
                float g[4], a[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) g[i] = Gs[q][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) a[j] = As[q][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) d[i][j] = fmaf(g[i], a[j], d[i][j]);
            }
            __syncthreads();
        }
        const int kb = kt0 + tx * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int n = n0 + ty * 4 + i;
            if (n >= N || kb >= K) continue;
            const float4 e = eps4(kk.key, kk.step, kk.s0 + s, L.t_w, n, kb >> 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                am[i][j] += d[i][j];
                ar[i][j] = fmaf(d[i][j], eps_get(e, j), ar[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int n = n0 + ty * 4 + i;
        if (n >= N) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = kt0 + tx * 4 + j;
            if (k >= K) continue;
            if (part) {
                const int64_t nk = (int64_t)N * K, o = (int64_t)n * K + k;
                part[(int64_t)blockIdx.z * 2 * nk + o] = scale * am[i][j];
                part[(int64_t)blockIdx.z * 2 * nk + nk + o] = scale * ar[i][j];
            } else {
                const int64_t o = L.off_w + (int64_t)n * K + k;
                acc_mu[o] += scale * am[i][j];
                acc_rho[o] += scale * ar[i][j];
            }
        }
    }
}

void launch_wgrad_fp32(const SampledLayer& L, const SampleKeys& k, int S, int B, const float* G,
                       int64_t strideG, const float* A, int64_t strideA, float scale,
                       float* acc_mu, float* acc_rho, cudaStream_t st, float* part, int64_t part_cap) {
    const int tiles = ((L.K + TB - 1) / TB) * ((L.N + TB - 1) / TB);
    int nsplit = 1;
    if (part) {  // enough row splits for ≈ 2 blocks per SM, within the scratch capacity
        nsplit = std::max(1, std::min({(2 * kNumSMs + tiles - 1) / tiles, (B + TK - 1) / TK,
                                       (int)(part_cap / (2 * (int64_t)L.N * L.K))}));
    }
    const int rows_per = ((B + nsplit - 1) / nsplit + TK - 1) / TK * TK;
    nsplit = (B + rows_per - 1) / rows_per;
    dim3 grid((L.K + TB - 1) / TB, (L.N + TB - 1) / TB, nsplit);
    wgrad_fp32_kernel<<<grid, 256, 0, st>>>(L, k, S, B, G, strideG, A, strideA, scale, acc_mu,
                                            acc_rho, rows_per, nsplit > 1 ? part : nullptr);
    if (nsplit > 1) launch_wgrad_split_reduce(part, nsplit, (int64_t)L.N * L.K, L.off_w, acc_mu, acc_rho, st);
}

// Bias gradient in two deterministic phases. parts[s][p][n] are fp32 partial column sums
// of the layer's output gradient (B rows in FP32 mode; 32-row chunks written by the BF16
// dgrad epilogue; the loss head's fp32 seed for the last layer).
//   phase A: db[s][n] = Σ_p parts[s][p][n]
//   phase B: acc_μ[b_n] += scale·Σ_s db[s][n];  acc_ρ[b_n] += scale·Σ_s db[s][n]·ε_s(t_b, 0, n)
constexpr int kBiasGroups = 32;  // at most; a launch uses G = blockDim.x / 32 part groups
__global__ void __launch_bounds__(32 * kBiasGroups)
    bias_reduce_kernel(SampledLayer L, SampleKeys kk, const float* __restrict__ parts, int nparts, int ldp,
                       int64_t strideS, int S, float* __restrict__ db) {
    __shared__ float red[kBiasGroups][33];
    const int G = blockDim.x >> 5;
    const int tx = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + tx, s = blockIdx.y;
    float acc = 0.0f;
    if (n < L.N) {  // group g: parts g, g+G, … (fixed order ⇒ deterministic)
        const float* p = parts + s * strideS + n;
        float a0 = 0.0f, a1 = 0.0f;
        int i = g;
        for (; i + G < nparts; i += 2 * G) {
            a0 += __ldg(p + (int64_t)i * ldp);
            a1 += __ldg(p + (int64_t)(i + G) * ldp);
        }
        if (i < nparts) a0 += __ldg(p + (int64_t)i * ldp);
        acc = a0 + a1;
    }
    red[g][tx] = acc;
    __syncthreads();
    if (g == 0 && n < L.N) {
        float t = 0.0f;
        for (int j = 0; j < G; ++j) t += red[j][tx];
        db[(int64_t)s * L.N + n] = t;
        db[(int64_t)(S + s) * L.N + n] = t * eps1(kk.key, kk.step, kk.s0 + s, L.t_b, 0, n);
    }
}

// Both phases in one launch for S ≤ 8 samples: the S blocks of a column block form a
// thread-block cluster (1 × S), each computes its sample's Σ_p as phase A does and leaves
// (t_s, t_s·ε_s) in its shared memory; the cluster's block 0 reads them over DSMEM in sample
// order and updates acc (fixed order ⇒ deterministic). Saves the phase-B launch (the ViT step
// has 54 bias tensors, each ≈ 4 µs of launch-bound phase B).
__global__ void __launch_bounds__(32 * kBiasGroups)
    bias_reduce_acc_cluster_kernel(SampledLayer L, SampleKeys kk, const float* __restrict__ parts, int nparts,
                                   int ldp, int64_t strideS, float scale, float* __restrict__ acc_mu,
                                   float* __restrict__ acc_rho) {
    namespace cg = cooperative_groups;
    __shared__ float red[kBiasGroups][33];
    __shared__ float out[2][32];
    cg::cluster_group cluster = cg::this_cluster();
    const int G = blockDim.x >> 5;
    const int tx = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + tx, s = blockIdx.y;
    float acc = 0.0f;
    if (n < L.N) {  // group g: parts g, g+G, … (fixed order)
        const float* p = parts + s * strideS + n;
        float a0 = 0.0f, a1 = 0.0f;
        int i = g;
        for (; i + G < nparts; i += 2 * G) {
            a0 += __ldg(p + (int64_t)i * ldp);
            a1 += __ldg(p + (int64_t)(i + G) * ldp);
        }
        if (i < nparts) a0 += __ldg(p + (int64_t)i * ldp);
        acc = a0 + a1;
    }
    red[g][tx] = acc;
    __syncthreads();
    if (g == 0) {
        float t = 0.0f;
        for (int j = 0; j < G; ++j) t += red[j][tx];
        out[0][tx] = t;
        out[1][tx] = n < L.N ? t * eps1(kk.key, kk.step, kk.s0 + s, L.t_b, 0, n) : 0.0f;
    }
    cluster.sync();
    if (cluster.block_rank() == 0 && g == 0 && n < L.N) {
        float m = 0.0f, r = 0.0f;
        for (unsigned b = 0; b < cluster.num_blocks(); ++b) {
            m += *cluster.map_shared_rank(&out[0][tx], b);
            r += *cluster.map_shared_rank(&out[1][tx], b);
        }
        acc_mu[L.off_b + n] += scale * m;
        acc_rho[L.off_b + n] += scale * r;
    }
    cluster.sync();  // the other blocks' shared memory stays alive until block 0 has read it
}

// phase B: 32 features × 8 sample groups per block, fixed-order smem combine (deterministic)
__global__ void bias_acc_kernel(SampledLayer L, int S, const float* __restrict__ db, float scale,
                                float* __restrict__ acc_mu, float* __restrict__ acc_rho) {
    __shared__ float red[2][8][33];
    const int tx = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + tx;
    float am = 0.0f, ar = 0.0f;
    if (n < L.N)
        for (int s = g; s < S; s += 8) {
            am += db[(int64_t)s * L.N + n];
            ar += db[(int64_t)(S + s) * L.N + n];
        }
    red[0][g][tx] = am;
    red[1][g][tx] = ar;
    __syncthreads();
    if (g == 0 && n < L.N) {
        float m = 0.0f, r = 0.0f;
        for (int i = 0; i < 8; ++i) {
            m += red[0][i][tx];
            r += red[1][i][tx];
        }
        acc_mu[L.off_b + n] += scale * m;
        acc_rho[L.off_b + n] += scale * r;
    }
}

// Grouped form (all layers of the MLP step in two launches instead of two per layer): the
// same per-layer arithmetic and summation order as bias_reduce_kernel / bias_acc_kernel.
__global__ void __launch_bounds__(32 * kBiasGroups)
    bias_reduce_grouped_kernel(const BiasGroup g, SampleKeys kk, int S, float* __restrict__ db_base) {
    __shared__ float red[kBiasGroups][33];
    int l = 0;
    while (l + 1 < g.n && (int)blockIdx.x >= g.blk_base[l + 1]) ++l;
    const SampledLayer& L = g.L[l];
    const int nparts = g.nparts[l], ldp = g.ldp[l];
    float* db = db_base + g.db_off[l];
    const int G = blockDim.x >> 5;
    const int tx = threadIdx.x & 31, gi = threadIdx.x >> 5;
    const int n = (blockIdx.x - g.blk_base[l]) * 32 + tx, s = blockIdx.y;
    float acc = 0.0f;
    if (n < L.N) {
        const float* p = g.parts[l] + s * g.strideS[l] + n;
        float a0 = 0.0f, a1 = 0.0f;
        int i = gi;
        for (; i + G < nparts; i += 2 * G) {
            a0 += __ldg(p + (int64_t)i * ldp);
            a1 += __ldg(p + (int64_t)(i + G) * ldp);
        }
        if (i < nparts) a0 += __ldg(p + (int64_t)i * ldp);
        acc = a0 + a1;
    }
    red[gi][tx] = acc;
    __syncthreads();
    if (gi == 0 && n < L.N) {
        float t = 0.0f;
        for (int j = 0; j < G; ++j) t += red[j][tx];
        db[(int64_t)s * L.N + n] = t;
        db[(int64_t)(S + s) * L.N + n] = t * eps1(kk.key, kk.step, kk.s0 + s, L.t_b, 0, n);
    }
}

__global__ void bias_acc_grouped_kernel(const BiasGroup g, int S, const float* __restrict__ db_base,
                                        float scale, float* __restrict__ acc_mu,
                                        float* __restrict__ acc_rho) {
    __shared__ float red[2][8][33];
    int l = 0;
    while (l + 1 < g.n && (int)blockIdx.x >= g.blk_base[l + 1]) ++l;
    const SampledLayer& L = g.L[l];
    const float* db = db_base + g.db_off[l];
    const int tx = threadIdx.x & 31, gi = threadIdx.x >> 5;
    const int n = (blockIdx.x - g.blk_base[l]) * 32 + tx;
    float am = 0.0f, ar = 0.0f;
    if (n < L.N)
        for (int s = gi; s < S; s += 8) {
            am += db[(int64_t)s * L.N + n];
            ar += db[(int64_t)(S + s) * L.N + n];
        }
    red[0][gi][tx] = am;
    red[1][gi][tx] = ar;
    __syncthreads();
    if (gi == 0 && n < L.N) {
        float m = 0.0f, r = 0.0f;
        for (int i = 0; i < 8; ++i) {
            m += red[0][i][tx];
            r += red[1][i][tx];
        }
        acc_mu[L.off_b + n] += scale * m;
        acc_rho[L.off_b + n] += scale * r;
    }
}

void launch_bias_grad_grouped(BiasGroup g, const SampleKeys& k, int S, float scale,
                              float* db_scratch, float* acc_mu, float* acc_rho, cudaStream_t st) {
    int blocks = 0, maxp = 1;
    int64_t off = 0;
    for (int l = 0; l < g.n; ++l) {
        g.blk_base[l] = blocks;
        g.db_off[l] = off;
        blocks += (g.L[l].N + 31) / 32;
        off += (int64_t)2 * S * g.L[l].N;
        maxp = std::max(maxp, g.nparts[l]);
    }
    int G = 1;
    while (G < kBiasGroups && G < maxp) G <<= 1;
    bias_reduce_grouped_kernel<<<dim3(blocks, S), 32 * G, 0, st>>>(g, k, S, db_scratch);
    bias_acc_grouped_kernel<<<blocks, 256, 0, st>>>(g, S, db_scratch, scale, acc_mu, acc_rho);
}

int launch_bias_grad(const SampledLayer& L, const SampleKeys& k, int S, const float* parts,
                     int nparts, int ldp, int64_t strideS, float scale, float* db_scratch,
                     float* acc_mu, float* acc_rho, cudaStream_t st) {
    dim3 grid((L.N + 31) / 32, S);
    int G = 1;  // part groups per block: enough for the part count (≤ 32), fewer threads when few parts
    while (G < kBiasGroups && G < nparts) G <<= 1;
    if (S >= 1 && S <= 8) {  // one launch: the S samples of a column block as a thread-block cluster
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(32 * G);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = (unsigned)S;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, bias_reduce_acc_cluster_kernel, L, k, parts, nparts, ldp, strideS, scale, acc_mu,
                               acc_rho) == cudaSuccess)
            return 1;
        (void)cudaGetLastError();  // cluster launch refused: the two-phase form below
    }
    bias_reduce_kernel<<<grid, 32 * G, 0, st>>>(L, k, parts, nparts, ldp, strideS, S, db_scratch);
    bias_acc_kernel<<<(L.N + 31) / 32, 256, 0, st>>>(L, S, db_scratch, scale, acc_mu, acc_rho);
    return 2;
}

// Many rows (the ViT's token rows): first each 64-row chunk is summed in row order into
// chunk[s][q][n] (one thread per (chunk, column), every chunk of a sample in parallel), then the
// two-phase reduction above runs on the chunk sums — the same fixed order every call.
__global__ void bias_rows_chunk_kernel(const float* __restrict__ parts, int nrows, int ldp, int64_t strideS, int N,
                                       int nchunks, float* __restrict__ chunk) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x, q = blockIdx.y, s = blockIdx.z;
    if (n >= N) return;
    const float* p = parts + s * strideS + (int64_t)q * 64 * ldp + n;
    const int r1 = min(64, nrows - q * 64);
    float a0 = 0.f, a1 = 0.f;
    int r = 0;
    for (; r + 1 < r1; r += 2) {
        a0 += __ldg(p + (int64_t)r * ldp);
        a1 += __ldg(p + (int64_t)(r + 1) * ldp);
    }
    if (r < r1) a0 += __ldg(p + (int64_t)r * ldp);
    chunk[((int64_t)s * nchunks + q) * N + n] = a0 + a1;
}

int launch_bias_grad_rows(const SampledLayer& L, const SampleKeys& k, int S, const float* parts, int nrows, int ldp,
                          int64_t strideS, float scale, float* scratch, int64_t scratch_cap, float* db_scratch,
                          float* acc_mu, float* acc_rho, cudaStream_t st) {
    const int nchunks = (nrows + 63) / 64;
    if (nrows <= 512 || !scratch || (int64_t)S * nchunks * L.N > scratch_cap)
        return launch_bias_grad(L, k, S, parts, nrows, ldp, strideS, scale, db_scratch, acc_mu, acc_rho, st);
    bias_rows_chunk_kernel<<<dim3((L.N + 127) / 128, nchunks, S), 128, 0, st>>>(parts, nrows, ldp, strideS, L.N,
                                                                               nchunks, scratch);
    return 1 + launch_bias_grad(L, k, S, scratch, nchunks, L.N, (int64_t)nchunks * L.N, scale, db_scratch, acc_mu,
                                acc_rho, st);
}

}  // namespace bnn
