// kernels.cuh — launcher declarations of libbnn's CUDA kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "eps.cuh"

namespace bnn {

// One sampled layer: W_s = μ + σ ⊙ ε_s over tensor t_w ([N, K]) and bias t_b ([1, N]).
struct SampledLayer {
    const float* mu;     // full μ vector
    const float* sigma;  // full σ = softplus(ρ) vector (written once per step by K7)
    int64_t off_w, off_b;
    int N, K;            // rows (outputs), cols (fan-in)
    uint32_t t_w, t_b;
};

// MC dropout of one hidden layer (R25): forward kernels multiply the
// post-ReLU value by keep·inv_keep; dgrad kernels scale the masked gradient by inv_keep.
struct DropArgs {
    int on;
    uint32_t p24;     // drop threshold in units of 2^-24
    float inv_keep;   // 1 / (1 − p)
    int layer;        // hidden-layer index of the mask key
    int b_off;        // global index of the rank's first example
};

struct SampleKeys {
    EpsKey key;
    uint32_t step;
    uint32_t s0;  // global index of the first sample of the chunk
};

// ---------------------------------------------------------------- K7 / K8 / K6 / K10 / K1
void launch_sigma(const float* rho, float* sigma, int64_t n, cudaStream_t st);
// grad_μ, grad_ρ, KL block partials (double), then loss = acc[2P] + KL/D
// loss[0] = L_data + KL/D, loss[1] = KL
void launch_finalize(int mcd, const float* mu, const float* rho, const float* acc_mu,
                     const float* acc_rho, const float* Ldata, int64_t P, double D,
                     float* grad_mu, float* grad_rho, double* kl_partials, int n_part,
                     float* loss, cudaStream_t st);
int finalize_partials_count(int64_t P);
// K8 + fused Adam: μ, ρ and the moments updated in place; grads optional
struct AdamHyper {
    float lr, beta1, beta2, eps;
    float omb1, omb2;  // 1 − β1, 1 − β2
    float bc1, bc2;    // 1 − β1^t, 1 − β2^t (host, double precision, rounded once)
};
void launch_finalize_adam(float* mu, float* rho, const float* acc_mu, const float* acc_rho,
                          const float* Ldata, int64_t P, double D, const AdamHyper& h,
                          float* m_mu, float* v_mu, float* m_rho, float* v_rho, float* grad_mu,
                          float* grad_rho, double* kl_partials, int n_part, float* loss,
                          cudaStream_t st);

// loss head on logits [S][B][O] fp32: writes dZ (unscaled gradient seed) as fp32 or bf16 with
// row stride ldg, and per-(s,b) loss values.
void launch_loss_head(const float* logits, int S, int B, int O, int loss_kind,
                      const int32_t* ycls, const float* yreg, void* dz, int ldg, bool dz_bf16,
                      float* lossrow, float* dz_f32, cudaStream_t st);
// exact aggregation: loss of the mean prediction over the S samples
// loss_kind 0 CE, 1 MSE, 2 Gaussian NLL of the predictive (stats: Welford mean, M2 per output;
// n_prev = samples already accumulated by earlier chunks)
void launch_mean_stats(const float* logits, int Sc, int B, int O, int loss_kind,
                       const int32_t* ycls, float* stats, int n_prev, cudaStream_t st);
void launch_mean_merge(const float* gathered, int world, int G, int g, int64_t n, float* out,
                       int gnll_O, int n_rank, cudaStream_t st);
void launch_mean_loss_head(const float* logits, int S, int B, int O, int loss_kind,
                           const int32_t* ycls, const float* yreg, const float* gstats,
                           int S_glob, void* dz, int ldg, bool dz_bf16, float* dz_f32,
                           cudaStream_t st);
void launch_mean_loss_value(const float* gstats, int B, int O, int loss_kind, const float* yreg,
                            int S_glob, float scale, float* acc_slot, cudaStream_t st);
// acc[2P] += scale · Σ lossrow[0..n) in fixed order
void launch_loss_reduce(const float* lossrow, int n, float scale, float* acc_slot,
                        cudaStream_t st);
void launch_eps_fill(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r0,
                     uint32_t nr, uint32_t c0, uint32_t nc, float* out, cudaStream_t st);
void launch_eps_table(int which, float* out, cudaStream_t st);
void launch_eps_bench(uint64_t n4, uint64_t seed, float* sink, int grid, cudaStream_t st);
// predict: probabilities/outputs [S][B][O] → local mean and M2 (two-pass)
void launch_predict_stats(const float* logits, int S, int B, int O, int loss_kind, float* mean,
                          float* m2, cudaStream_t st);
// ordered Chan merge of per-rank (mean, M2, n) [R][BO] → mean, var (÷ total n)
void launch_predict_merge(const float* means, const float* m2s, const float* counts, int R,
                          int BO, float* mean, float* var, cudaStream_t st);
// x fp32 [B][K] → bf16 [B][ldx] (zero padding of columns K..ldx)
void launch_bf16_to_f32(const void* x, int64_t n, float* y, cudaStream_t st);
void launch_to_bf16(const float* x, int B, int K, int ldx, void* out, cudaStream_t st);

// ---------------------------------------------------------------- K11: FP32 SIMT sampled GEMMs
// Z[s][b][n] = act(Σ_k A[s][b][k]·W_s[n][k] + b_s[n]) for s in [0, S), b in [0, B).
void launch_fwd_fp32(const SampledLayer& L, const SampleKeys& k, const DropArgs& d, int S, int B, const float* A,
                     int64_t strideA, float* Z, int64_t strideZ, bool relu, cudaStream_t st);
// dA[s][b][k] = (Σ_n G[s][b][n]·W_s[n][k]) · 1[A[s][b][k] > 0]
void launch_dgrad_fp32(const SampledLayer& L, const SampleKeys& k, const DropArgs& d, int S, int B, const float* G,
                       int64_t strideG, const float* Aprev, int64_t strideA, float* dA,
                       int64_t strideD, cudaStream_t st);
// acc_μ[n][k] += scale·Σ_s dW_s[n][k]; acc_ρ[n][k] += scale·Σ_s dW_s[n][k]·ε_s[n][k] with
// dW_s = Σ_b G[s][b][n]·A[s][b][k]; plus the bias: db_s[n] = Σ_b G[s][b][n].
// part (optional, capacity part_cap floats): split the B rows over blocks (the ViT's token rows)
// with scaled partials [split][μ|ρ][N·K] reduced in split order into acc (deterministic).
void launch_wgrad_fp32(const SampledLayer& L, const SampleKeys& k, int S, int B, const float* G,
                       int64_t strideG, const float* A, int64_t strideA, float scale,
                       float* acc_mu, float* acc_rho, cudaStream_t st, float* part = nullptr,
                       int64_t part_cap = 0);
void launch_wgrad_split_reduce(const float* part, int nsplit, int64_t n, int64_t off, float* acc_mu,
                               float* acc_rho, cudaStream_t st);
// bias gradient from fp32 partial column sums parts[s][p][n] (p < nparts, row pitch ldp)
// all bias tensors of up to 4 layers in two launches (per-layer parts as launch_bias_grad;
// db_scratch holds 2·S·N_l floats per layer, consecutively)
constexpr int kMaxBiasGroup = 4;
struct BiasGroup {
    SampledLayer L[kMaxBiasGroup];
    const float* parts[kMaxBiasGroup];
    int nparts[kMaxBiasGroup], ldp[kMaxBiasGroup];
    int64_t strideS[kMaxBiasGroup];
    int blk_base[kMaxBiasGroup];
    int64_t db_off[kMaxBiasGroup];
    int n;
};
void launch_bias_grad_grouped(BiasGroup g, const SampleKeys& k, int S, float scale,
                              float* db_scratch, float* acc_mu, float* acc_rho, cudaStream_t st);
int launch_bias_grad(const SampledLayer& L, const SampleKeys& k, int S, const float* parts,
                      int nparts, int ldp, int64_t strideS, float scale, float* db_scratch,
                      float* acc_mu, float* acc_rho, cudaStream_t st);
// the same for many rows (nrows > 512): 64-row chunk sums into `scratch` first (capacity in floats)
int launch_bias_grad_rows(const SampledLayer& L, const SampleKeys& k, int S, const float* parts, int nrows, int ldp,
                           int64_t strideS, float scale, float* scratch, int64_t scratch_cap, float* db_scratch,
                           float* acc_mu, float* acc_rho, cudaStream_t st);

}  // namespace bnn
