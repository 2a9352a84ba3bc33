/*
 * bnn.h — C ABI of libbnn.so, the B200-native Bayes-by-backprop ELBO step with sampling
 * parallelism (arXiv 2604.04736, "Sampling Parallelism for Fast and Efficient Bayesian
 * Learning").
 *
 * The library computes, for a mean-field Gaussian BNN with variational parameters (μ, ρ),
 * σ = softplus(ρ), one minibatch (x, y), S Monte-Carlo samples, a 64-bit seed and a step
 * counter:
 *     w_s    = μ + σ ⊙ ε_s,  ε_s from EPS-v1 (docs/EPS.md)       PAPER.md:158-159 (Alg. 1 l.5-6)
 *     ŷ_s    = ForwardPass(x, w_s)                               PAPER.md:160 (Alg. 1 l.7)
 *     L_data = (1/S) Σ_s Loss(ŷ_s, y)                            PAPER.md:162 (Alg. 1 l.9)
 *     KL     = ½ Σ_i (σ_i² + μ_i² − 1 − log σ_i²)                PAPER.md:163 (Alg. 1 l.10)
 *     loss   = L_data + KL / |D|                                 PAPER.md:164 (Alg. 1 l.11)
 *     grad_μ = ∂loss/∂μ,  grad_ρ = ∂loss/∂ρ                      PAPER.md:165 (Alg. 1 l.12)
 * with the S samples (and optionally the batch) sharded over the ranks of one node and a
 * single SUM-allreduce of the gradient partials (§4.1, Alg. 2
 * PAPER.md:250-264; hybrid sample×data grid PAPER.md:283-295, §4.2). The optimizer step
 * (Alg. 1 l.13) is the caller's, or fused into the finalize pass (bnn_elbo_step_adam,
 * Adam). Readings of points the paper leaves open are DESIGN.md §2.
 *
 * Conventions for every entry point:
 *  - Return value: BNN_OK (0) or a bnn_status code; bnn_last_error() names the violated
 *    invariant. Entry points never abort the process.
 *  - Pointers named *_dev are CUDA device pointers on cfg.device; *_host are host pointers.
 *    Unless stated, tensors are dense, row-major, 16-byte aligned (256-byte preferred).
 *  - The caller owns every tensor passed in. The library owns its workspace (allocated in
 *    bnn_init, never inside a step), its NCCL communicator and its CUDA streams/events.
 *  - All device work is enqueued on cfg.stream (NULL: the legacy default stream); calls
 *    return after enqueue unless a *_host output is requested, which synchronises.
 *  - A bnn_ctx is used by one host thread at a time.
 *  - There is no CPU fallback: without a usable sm_100 device bnn_init fails with
 *    BNN_ERR_CUDA.
 *
 * Parameter layout: a flat fp32 vector of n_params entries; for each layer
 * l in model order, weight tensor t = 2l viewed as [rows = c_out, cols = kh·kw·c_in]
 * (OHWI, c_in fastest; a linear layer is kh = kw = 1), then bias tensor t = 2l+1 viewed as
 * [1, c_out]. μ, ρ, grad_μ and grad_ρ all use this layout.
 */
#ifndef BNN_H_
#define BNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BNN_ABI_VERSION 3  /* 3: bnn_config.comm_timeout_ms, bnn_sync (non-blocking communicator, bucketed exchange);
                              2: bnn_model_desc.method / .dropout_p (MC dropout), Adam, mean-aggregation entry points */

typedef enum {
    BNN_OK = 0,
    BNN_ERR_CONFIG = 2,  /* invalid model/config/shape/alignment (SPEC.md:426-428 invariants) */
    BNN_ERR_COMM = 3,    /* NCCL error or timeout */
    BNN_ERR_NUMERIC = 4, /* non-finite loss (only checked when the loss is read on the host) */
    BNN_ERR_CUDA = 5     /* CUDA runtime/driver error, or no sm_100 device */
} bnn_status;

enum { BNN_MODEL_MLP = 0, BNN_MODEL_RESNET18 = 1, BNN_MODEL_VIT = 2 };
/* BNN_LOSS_CE / _MSE: L_data = (1/S) Σ_s Loss(ŷ_s, y), the per-sample average of Alg. 1 l.9
 * (PAPER.md:162). BNN_LOSS_CE_MEAN / _MSE_MEAN: exact aggregation (§4.1;
 * SURVEY.md §8(f) f1), the loss of the MEAN prediction — CE of the arithmetic mean of the
 * class probabilities over the S samples, MSE of the mean output. The mean
 * needs every sample group's statistic before any backward: bnn_elbo_step exchanges it with
 * one extra allgather between forward and backward; virtual ranks use bnn_mean_stats +
 * bnn_elbo_partial_mean. MLP and ResNet models, both precisions. */
/* BNN_LOSS_GNLL_MEAN: Gaussian NLL of the predictive distribution, the two-parameter case of
 * P:281 ("Gaussian negative log-likelihood"; mean and population variance of the S
 * predictions per output, variance floor 1e-6, R24): fp32 targets [B, outputs];
 * statistic per rank = Welford (mean, M2) of its samples, merged by Chan's update. MLP models,
 * precision FP32 only (BNN_ERR_CONFIG otherwise: bf16-rounded predictions perturb the sample
 * variance the gradient divides by beyond the BF16 tolerance). */
enum { BNN_LOSS_CE = 0, BNN_LOSS_MSE = 1, BNN_LOSS_CE_MEAN = 2, BNN_LOSS_MSE_MEAN = 3,
       BNN_LOSS_GNLL_MEAN = 4 };
enum { BNN_PREC_FP32 = 0, BNN_PREC_BF16 = 1 };
enum { BNN_MODE_SAMPLE_SHARDED = 0, BNN_MODE_DATA_SHARDED = 1, BNN_MODE_HYBRID = 2 };
enum { BNN_AUG_NONE = 0, BNN_AUG_PER_SAMPLE = 1 };
/* BNN_METHOD_MCD: Monte Carlo dropout (use case 2
 * P:318-320; R25): the weights are μ (ρ is ignored, grad_rho = 0, no prior term),
 * a "sample" is one draw of inverted-dropout masks on every hidden activation, keyed by
 * (seed, step, global sample, layer, global example, unit). MLP models only. */
enum { BNN_METHOD_VI = 0, BNN_METHOD_MCD = 1 };

/* Model description.
 *  MLP:      widths[0] = input features, widths[n_widths-1] = outputs; ReLU between layers.
 *  RESNET18: CIFAR ResNet-18 topology without BatchNorm (reading R12): 3×3 stem,
 *            4 stages × 2 BasicBlocks of widths base_width·{1,2,4,8}, stride-2 1×1
 *            projections, global average pool, linear head to n_classes. Input NHWC fp32. */
typedef struct bnn_model_desc {
    int32_t kind;
    int32_t n_widths;
    int32_t widths[16];
    int32_t in_h, in_w, in_c;
    int32_t n_classes;
    int32_t base_width;
    int32_t loss; /* BNN_LOSS_CE (labels int32 in [0, n_classes); an out-of-range label gives a
                     NaN loss, i.e. BNN_ERR_NUMERIC when the loss is read, never an out-of-bounds
                     read) | BNN_LOSS_MSE (targets fp32 [B, outputs]) */
    int32_t method;   /* BNN_METHOD_VI (Bayes by backprop, default) | BNN_METHOD_MCD */
    float dropout_p;  /* MCD: drop probability of every hidden unit, 0 ≤ p < 1 */
    /* BNN_MODEL_VIT: in_h × in_w × in_c images (NHWC fp32),
     * patch × patch patches, width dim, `heads` attention heads, `depth` pre-norm encoder
     * layers with an MLP of width mlp, n_classes outputs, loss BNN_LOSS_CE; dim % heads == 0,
     * dim % 4 == 0, dim ≥ 32, 1 + (in_h/patch)·(in_w/patch) ≤ 68 tokens, dim/heads ≤ 68; FP32
     * (SIMT) or BF16 (projections on tcgen05, attention on the TF32 warp MMA; patch·patch·in_c,
     * dim, mlp multiples of 8; B_loc == max_B_loc). Violations: BNN_ERR_CONFIG at bnn_create.
     * bnn_predict and the *_MEAN losses are not available for it (BNN_ERR_CONFIG).
     * Tensor order and shapes: oracle/vit_oracle.c header / DESIGN.md §3 (every tensor,
     * LayerNorm g/b, cls and pos included, is variational). */
    int32_t patch, dim, heads, depth, mlp;
} bnn_model_desc;

/* Run configuration. Rank r of world P = K·G is sample group k = r / G, data group
 * g = r % G; it owns global samples [k·S/K, (k+1)·S/K) and global examples
 * [g·B/G, (g+1)·B/G). SAMPLE_SHARDED forces K = world, G = 1;
 * DATA_SHARDED forces K = 1, G = world; HYBRID takes K, G as given. */
typedef struct bnn_config {
    int32_t precision;        /* BNN_PREC_FP32 (SIMT fp32, parity mode) | BNN_PREC_BF16 (tcgen05) */
    int32_t mode;             /* BNN_MODE_* */
    int32_t K, G;             /* HYBRID grid; ignored otherwise */
    int32_t rank, world;
    const uint8_t* nccl_uid;  /* 128-byte id from bnn_get_unique_id on rank 0 (broadcast by the
                                 caller), or NULL: no communicator. With NULL and world > 1 the
                                 context is a "virtual rank": use bnn_elbo_partial/bnn_finalize. */
    int32_t max_B_loc;        /* largest per-rank batch a step will pass. FP32 contexts and BF16
                                 MLP contexts accept any 0 < B_loc <= max_B_loc per step (the BF16
                                 MLP re-encodes its TMA descriptors on the host when B_loc changes);
                                 BF16 ResNet contexts lay out descriptors, scratch splits and grids
                                 for max_B_loc and require B_loc == max_B_loc (BNN_ERR_CONFIG) */
    int32_t max_S_loc;        /* largest per-rank sample count a step will use */
    int32_t sample_chunk;     /* samples processed together (0 = all local samples) */
    int32_t aug;              /* BNN_AUG_NONE | BNN_AUG_PER_SAMPLE (images only; docs/EPS.md §4) */
    double dataset_size;      /* |D| of PAPER.md:164, > 0 */
    int32_t device;           /* CUDA device ordinal */
    void* stream;             /* cudaStream_t; NULL = the legacy default stream */
    int32_t comm_timeout_ms;  /* > 0: a collective (or the communicator's init) that has not
                                 completed after this long, or an NCCL async error, aborts the
                                 communicator (ncclCommAbort) and the call returns BNN_ERR_COMM
                                 (SPEC.md:397, :733). 0: env BNN_COMM_TIMEOUT_MS, else 600000.
                                 Checked wherever the library waits on the host: bnn_init, the
                                 loss read of bnn_elbo_step*, bnn_sync. */
} bnn_config;

typedef struct bnn_tensor_info {
    int64_t offset;  /* element offset in the flat parameter vector */
    int32_t rows;    /* c_out (weights) or 1 (biases) */
    int32_t cols;    /* kh·kw·c_in (weights) or c_out (biases) */
    int32_t t;       /* tensor index used by EPS-v1 keys */
    int32_t is_bias;
} bnn_tensor_info;

typedef struct bnn_ctx bnn_ctx;

/* NCCL unique id for a new communicator; call on rank 0 and broadcast the 128 bytes. */
int bnn_get_unique_id(uint8_t out[128]);

/* Validate model and config, select the device, build the layer graph and parameter
 * layout, allocate all workspace, create the NCCL communicator (if nccl_uid != NULL).
 * Errors: BNN_ERR_CONFIG (e.g. "world == K*G", "S mod K == 0" is checked per step),
 * BNN_ERR_CUDA (no sm_100 device / out of memory), BNN_ERR_COMM. */
int bnn_init(const bnn_model_desc* model, const bnn_config* cfg, bnn_ctx** out);

/* Parameter layout: *n_params total entries; up to max_infos tensor records written to
 * infos (may be NULL); *n_tensors receives the tensor count. */
int bnn_param_layout(bnn_ctx* ctx, int64_t* n_params, int32_t* n_tensors,
                     bnn_tensor_info* infos, int32_t max_infos);

/* One full ELBO step on this rank: σ prologue, (augmentation), per local
 * sample chunk: sampled forward, loss head, sampled backward with the sample-accumulating
 * wgrad epilogue; SUM-allreduce of [acc_μ | acc_ρ | L_data] over all ranks; finalize + KL.
 *   mu_dev, rho_dev        [n_params] fp32, identical on all ranks
 *   x_dev                  this rank's examples [B_loc, features] (MLP) or [B_loc, H, W, C]
 *                          NHWC (ResNet) fp32
 *   ycls_dev / yreg_dev    int32 [B_loc] labels (CE) or fp32 [B_loc, outputs] (MSE); the
 *                          other is NULL
 *   B_loc, B_global        per-rank and global batch (B_global == G·B_loc)
 *   S_global               global sample count (S_global mod K == 0, S_global/K ≤ max_S_loc)
 *   seed, step             EPS-v1 key and counter word (docs/EPS.md §1)
 *   loss_dev               device fp32 scalar (may be NULL)
 *   loss_host              if non-NULL, the loss is copied back (synchronises) and checked
 *                          for finiteness (BNN_ERR_NUMERIC)
 *   grad_mu_dev, grad_rho_dev  [n_params] fp32 outputs, identical on all ranks on return */
int bnn_elbo_step(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev, const float* x_dev,
                  const int32_t* ycls_dev, const float* yreg_dev, int32_t B_loc,
                  int32_t B_global, int32_t S_global, uint64_t seed, uint32_t step,
                  float* loss_dev, double* loss_host, float* grad_mu_dev, float* grad_rho_dev);

/* Same step with the minibatch in HOST memory (pinned recommended): x/y are copied into
 * library-owned device buffers on the ctx stream inside the call, and the loss is read
 * back into *loss_host (synchronises). The end-to-end path of bench.py. */
int bnn_elbo_step_host(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev,
                       const float* x_host, const int32_t* ycls_host, const float* yreg_host,
                       int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                       uint32_t step, double* loss_host, float* grad_mu_dev,
                       float* grad_rho_dev);

/* Layout of the gradient-partial ("acc") buffer exchanged by the allreduce: acc_μ at 0,
 * acc_ρ at *rho_offset (n_params rounded up to 64 so every segment is 256-byte aligned),
 * the L_data partial at *loss_offset; *total floats in all. */
int bnn_acc_layout(bnn_ctx* ctx, int64_t* rho_offset, int64_t* loss_offset, int64_t* total);

/* This rank's shard only, no collective and no finalize: writes acc_dev (bnn_acc_layout) =
 * [Σ_s dW_s | Σ_s dW_s ⊙ ε_s | L_data partial], each pre-scaled by the global 1/(S·B)
 * (reading R8). Summing the acc of every rank of a K×G grid and calling
 * bnn_finalize equals bnn_elbo_step. */
int bnn_elbo_partial(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev,
                     const float* x_dev, const int32_t* ycls_dev, const float* yreg_dev,
                     int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                     uint32_t step, float* acc_dev);

/* Finalize + KL (Alg. 1 l.10-12) from a summed acc buffer:
 *   grad_μ = acc_μ + μ/|D|;  grad_ρ = sigmoid(ρ)·(acc_ρ + (σ − 1/σ)/|D|);
 *   loss = acc[2P] + ½Σ(σ² + μ² − 1 − 2 ln σ)/|D|. */
int bnn_finalize(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev, const float* acc_dev,
                 float* loss_dev, float* grad_mu_dev, float* grad_rho_dev);

/* Exact aggregation, virtual-rank form (BNN_LOSS_*_MEAN only). bnn_mean_stats runs this
 * rank's sampled forward passes and writes its statistic: stats_dev[b·w + j] = Σ over the
 * rank's samples of p_{s,b,y_b} (CE, w = 1) or of ŷ_{s,b,j} (MSE, w = outputs), fp32, for its
 * B_loc examples; GNLL: w = 2·outputs, [mean (outputs) | M2 (outputs)] of the rank's samples.
 * Merging the stats of the K sample groups of a data group (bnn_mean_merge: the sum for CE /
 * MSE, Chan's update for GNLL) and passing the result to bnn_elbo_partial_mean yields this
 * rank's acc partial of the exact step (the data loss is counted by sample group 0). */
int bnn_mean_stats(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev, const float* x_dev,
                   const int32_t* ycls_dev, int32_t B_loc, int32_t B_global, int32_t S_global,
                   uint64_t seed, uint32_t step, float* stats_dev);
/* Merge of n_groups statistics stats_all [n_groups][B_loc·w] (rank order) into out [B_loc·w],
 * the same device merge bnn_elbo_step applies after its allgather; each group holds
 * S_global / n_groups samples. */
int bnn_mean_merge(bnn_ctx* ctx, const float* stats_all, int32_t n_groups, int32_t B_loc,
                   int32_t S_global, float* out);
int bnn_elbo_partial_mean(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev,
                          const float* x_dev, const int32_t* ycls_dev, const float* yreg_dev,
                          int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                          uint32_t step, const float* stats_global_dev, float* acc_dev);

/* Adam hyper-parameters of the fused optimizer step (PAPER.md:166 and
 * :265, Alg. 1 l.13 / Alg. 2 l.16 "Update μ and σ using optimizer (e.g., Adam)"; Kingma & Ba
 * Algorithm 1). Requires lr ≥ 0, 0 ≤ beta1, beta2 < 1, eps > 0, t ≥ 1 (BNN_ERR_CONFIG). */
typedef struct bnn_adam {
    float lr, beta1, beta2, eps;
    int32_t t; /* 1-based update count: bias corrections 1 − beta1^t, 1 − beta2^t */
} bnn_adam;

/* Finalize + KL + Adam in one pass over the parameters: the gradients of bnn_finalize are
 * formed in registers and, for θ ∈ {μ, ρ} with gradient g,
 *   m ← β1·m + (1−β1)·g;  v ← β2·v + (1−β2)·g²;  θ ← θ − lr·(m/(1−β1^t)) / (√(v/(1−β2^t)) + eps)
 * updates mu_dev, rho_dev and the four moment buffers in place (fp32 [n_params] each,
 * caller-owned, zero before the first update). The loss (and KL) are those of the parameters
 * BEFORE the update. grad_mu_dev / grad_rho_dev may be NULL (not written). */
int bnn_finalize_adam(bnn_ctx* ctx, float* mu_dev, float* rho_dev, const float* acc_dev,
                      const bnn_adam* adam, float* m_mu_dev, float* v_mu_dev, float* m_rho_dev,
                      float* v_rho_dev, float* loss_dev, float* grad_mu_dev, float* grad_rho_dev);

/* bnn_elbo_step whose finalize is bnn_finalize_adam: one training step (Alg. 1 l.4-13 /
 * Alg. 2 l.5-16) with μ, ρ and the moments updated in place on every rank (all ranks apply
 * the same update to the same allreduced gradient). Arguments as bnn_elbo_step and
 * bnn_finalize_adam. */
int bnn_elbo_step_adam(bnn_ctx* ctx, float* mu_dev, float* rho_dev, const float* x_dev,
                       const int32_t* ycls_dev, const float* yreg_dev, int32_t B_loc,
                       int32_t B_global, int32_t S_global, uint64_t seed, uint32_t step,
                       const bnn_adam* adam, float* m_mu_dev, float* v_mu_dev, float* m_rho_dev,
                       float* v_rho_dev, float* loss_dev, double* loss_host, float* grad_mu_dev,
                       float* grad_rho_dev);

/* Posterior predictive over S_global samples: per output element
 * the mean and the population variance (÷S) of softmax probabilities (CE) or outputs
 * (MSE). x_dev holds all B examples (predict is sample-sharded only); every rank returns
 * the full [B, outputs] mean_dev/var_dev after an allgather of per-rank (mean, M2, n). */
int bnn_predict(bnn_ctx* ctx, const float* mu_dev, const float* rho_dev, const float* x_dev,
                int32_t B, int32_t S_global, uint64_t seed, uint32_t step, float* mean_dev,
                float* var_dev);

/* EPS-v1 ε (docs/EPS.md) for tensor t, sample s, rows [r0, r0+nr), cols [c0, c0+nc):
 * out_dev[i·nc + j] = ε(seed, step, s, t, r0+i, c0+j). Stand-alone K1 kernel, used by the
 * bit-exactness tests. stream may be NULL (legacy default stream). */
int bnn_eps_fill(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r0,
                 uint32_t nr, uint32_t c0, uint32_t nc, float* out_dev, void* stream);

/* Every value of the EPS-v1 transform pieces (docs/EPS.md §3), for the exhaustive
 * bit-exactness test: which = 0 → out[k-1] = R = sqrt_rn(-2·LOG24(k·2^-24)), k = 1..2^24;
 * which = 1 / 2 → out[v] = cos / sin part of SINCOS2PI24(v), v = 0..2^24-1.
 * out_dev holds 2^24 floats. */
int bnn_eps_transform_table(int32_t which, float* out_dev, void* stream);

/* ε-throughput microbenchmark (the ALU roofline of DESIGN.md §4): generates n4·4 normals
 * with the same code as the fused kernels and reduces them into sink_dev[grid] instead of
 * storing them. */
int bnn_eps_bench(uint64_t n4, uint64_t seed, float* sink_dev, int32_t grid, void* stream);

/* Per-kernel-class device timing, measured with CUDA events on the ctx stream around each
 * launch while enabled (bench.py's roofline). names: comma-separated classes. */
int bnn_profile_enable(bnn_ctx* ctx, int32_t on);
int bnn_profile_read(bnn_ctx* ctx, char* names, int32_t names_cap, double* ms, int64_t* launches,
                     int32_t max_entries, int32_t* n_entries);

/* Test hook (ResNet contexts): copy the stored output (which = 0) or output gradient
 * (which = 1) of layer `layer` of the last step, [S_chunk][B][H][W][C] as fp32, into out_dev
 * (cap floats); *n_out receives the element count. Synchronises. */
int bnn_debug_layer_output(bnn_ctx* ctx, int32_t layer, int32_t which, float* out_dev,
                           int64_t cap, int64_t* n_out);

/* Number of kernels the library launched since bnn_init (bench.py's gpu_launches). */
int64_t bnn_launch_count(bnn_ctx* ctx);

/* Message for the last error on ctx (or the last context-free error if ctx is NULL). */
/* Wait on the host until everything enqueued on the context's stream (and its comm stream)
 * has completed, polling the communicator: a failed or silent peer returns BNN_ERR_COMM after
 * comm_timeout_ms (the communicator is aborted; bnn_destroy is the only valid call after it),
 * a CUDA error BNN_ERR_CUDA. Without a communicator: cudaStreamSynchronize. */
int bnn_sync(bnn_ctx* ctx);

/* Diagnostic: the number of NCCL groups (layer buckets, the tail with L_data included) the
 * last bnn_elbo_step* exchange issued; 0 without a communicator. */
int32_t bnn_comm_buckets(bnn_ctx* ctx);

const char* bnn_last_error(bnn_ctx* ctx);

void bnn_destroy(bnn_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BNN_H_ */
