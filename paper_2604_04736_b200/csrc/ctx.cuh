// ctx.cuh — private: the bnn_ctx state shared by the runtime translation units.
#pragma once
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <array>
#include <vector>

#include "../../include/bnn.h"
#include "kernels.cuh"
#include "kernels_conv.cuh"
#include "kernels_tc.cuh"

using namespace bnn;

namespace bnn_rt {
extern thread_local std::string g_last_error;

struct LayerDesc {
    int cin, cout, k, stride, pad;
    int64_t off_w, off_b;
    uint32_t t_w, t_b;
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D bf16 view [depth][rows][inner] with row pitch ld elements, box (64, box_rows, 1),
// 128-byte swizzle, zero fill out of bounds.
inline bool make_map(CUtensorMap* m, const void* base, int inner, int rows, int depth, int ld,
              int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)depth};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * rows};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// generic bf16 tensor map: rank ≤ 5, dims[0] contiguous, strides in bytes for dims 1..rank-1
inline bool make_map_nd(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                        const uint64_t* strides, const uint32_t* box, const uint32_t* estr = nullptr,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        bx[i] = box[i];
        es[i] = estr ? estr[i] : 1;  // traversal stride (a strided conv window), box counts raw elements
        if (i > 0) st[i - 1] = strides[i - 1];
    }
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, st, bx, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace bnn_rt
using namespace bnn_rt;

// ResNet graph (the CNN of C3–C5): every op is a fused conv (+bias, +residual, ReLU) or GAP.
struct RBuf {
    int H, W, C;
    float* val;
    float* grad;
};
struct ROp {
    int type;  // 0 conv, 1 global average pool
    int layer, src, dst, res, relu;
};

struct bnn_ctx {
    bnn_model_desc model{};
    bnn_config cfg{};
    std::vector<LayerDesc> layers;
    std::vector<int> widths;  // MLP widths
    int64_t P = 0, P_pad = 0, acc_total = 0;
    int O = 0;
    int K = 1, G = 1, kidx = 0, gidx = 0;
    int S_loc_max = 0, B_max = 0, chunk = 0;
    bool bf16 = false;
    int agg = 0;               // 1: loss of the mean prediction (BNN_LOSS_*_MEAN), SURVEY §8(f) f1
    int gnll = 0;              // agg with the Gaussian NLL of the predictive (mean, variance)
    int mcd = 0;               // MC dropout
    uint32_t p24 = 0;          // MCD drop threshold, units of 2^-24
    float inv_keep = 1.0f;
    DropArgs drop_for(int layer, bool on, int B) const {
        DropArgs d{};
        d.on = (mcd && on) ? 1 : 0;
        d.p24 = p24;
        d.inv_keep = inv_keep;
        d.layer = layer;
        d.b_off = gidx * B;
        return d;
    }
    int mkind() const { return gnll ? 2 : model.loss; }  // loss kind of the mean-statistic kernels
    int stat_w = 0;            // agg: statistic width per example (CE 1, MSE O)
    float* mstats = nullptr;   // agg: this rank's Σ_s statistic [B_max × stat_w]
    float* mstats_g = nullptr; // agg: merged over the sample groups
    float* mgather = nullptr;  // agg: allgather buffer [world × B_max × stat_w]
    cudaStream_t st = nullptr;
    bool own_stream = false;
    // side stream for the small kernels that overlap the wgrad GEMM (loss reduction, bias
    // gradients): forked from / joined into st with events; unused while profiling
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // second side stream (CNN bias gradients, beside the wgrad / ε-combine stream)
    cudaStream_t side2 = nullptr;
    cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
    ncclComm_t comm = nullptr;
    // gradient exchange (comm.cu): non-blocking communicator, comm stream, layer buckets
    cudaStream_t comm_st = nullptr;
    cudaEvent_t ev_comm_in = nullptr, ev_comm_out = nullptr;
    double comm_timeout_ms = 600000.0;
    bool comm_aborted = false;
    int64_t ar_bucket_bytes = 16 << 20;
    bool ar_enabled = false, ar_live = false, ar_live_used = false;
    int ar_top = -1, ar_buckets = 0;
    std::vector<char> ar_done;
    std::vector<std::array<cudaEvent_t, 2>> ar_ev;
    // workspace
    float* sigma = nullptr;
    float* acc = nullptr;
    double* kl_part = nullptr;
    int n_part = 0;
    float* lossbuf = nullptr;  // [0] loss, [1] KL
    float* lossrow = nullptr;
    float* logits = nullptr;
    std::vector<void*> act;    // act[l]: input of layer l (l ≥ 1)
    std::vector<int> ld;       // padded row pitch of width l
    std::vector<void*> grad;   // grad[l]: dℓ/dz of layer l output
    std::vector<float*> dbpart;  // BF16: fp32 32-row column sums of grad[l] (l < L-1)
    float* dz_f32 = nullptr;     // BF16: fp32 copy of the loss-head seed [S][B][O]
    float* db_scratch = nullptr; // [S][max N] per-sample bias gradients
    void* xb = nullptr;        // bf16 copy of the layer-0 input
    float* x_stage = nullptr;  // device copy of a host batch
    int32_t* ycls_stage = nullptr;
    float* yreg_stage = nullptr;
    float* p_mean = nullptr;
    float* p_m2 = nullptr;
    float* g_means = nullptr;
    float* g_m2s = nullptr;
    float* g_counts = nullptr;
    float* acc_scratch = nullptr;  // for bnn_elbo_step_host / predict helpers
    std::vector<RBuf> rbufs;       // ResNet activations / gradients, [S_chunk][B][H][W][C]
    std::vector<ROp> rops;
    int rlogits = -1;
    int64_t in_elems = 0;          // per-example input elements
    // BF16 ResNet state (parallel to rbufs / layers)
    struct RBf {
        __nv_bfloat16* val = nullptr;
        __nv_bfloat16* grad = nullptr;
        float* bpart = nullptr;    // fp32 bias-gradient partials of the buffer's producer
        uint32_t* mbits = nullptr; // ReLU bitmask [s][pixel][C/32] of a ReLU output (dgrad mask)
        int nparts = 0;
        int C_pad = 0;
        int64_t bpart_cap = 0;
    };
    std::vector<RBf> rbf;
    __nv_bfloat16* wscr = nullptr;  // W_s scratch of every conv layer for the sample chunk
    std::vector<size_t> wscr_off;   // per layer: element offset of its slot (forward writes, dgrad reads)
    float* wpart = nullptr;         // conv wgrad split partials (buffer 0)
    float* wpart2 = nullptr;        // buffer 1: consecutive layers alternate, so the ε combine of
                                    // one layer overlaps the wgrad GEMM of the next
    cudaStream_t side3 = nullptr;   // ε-combine stream
    cudaEvent_t ev_wg[2] = {nullptr, nullptr}, ev_comb[2] = {nullptr, nullptr}, ev_join3 = nullptr;
    std::vector<int> kpad, nsplit;  // per layer
    std::vector<int> wkpx;          // per layer: wgrad pixels per k-step (64 or 128)
    std::vector<CUtensorMap> cmap_w, cmap_wT, cmap_g;  // per layer
    std::vector<CUtensorMap> cmap_bf, cmap_bd;         // per layer: 5-D activation / dY windows
    std::vector<CUtensorMap> cmap_xw;                  // per layer: wgrad X windows (64 pixels)
    std::vector<CUtensorMap> cmap_a2f, cmap_a2d, cmap_w2, cmap_w64;  // conv2: 128-pixel A windows, W (n_tile rows)
    std::vector<char> tma_a2f, tma_a2d;
    float* bias_scr = nullptr;                         // sampled conv biases [layer][S][512]
    std::vector<cudaEvent_t> wgen_ev;                  // per layer: W_s slot written (side stream)
    std::vector<char> tma_fwd, tma_dgrad, tma_wgrad;   // stride-1 layers use them
    // Bayesian ViT (runtime_vit.cu): tensor table, activations per layer, gradient scratch
    struct VitTensor {
        int64_t off;
        int rows, cols;
    };
    struct VitAct {
        float *X = nullptr, *H1 = nullptr, *st1 = nullptr, *QKV = nullptr, *Att = nullptr, *O = nullptr,
              *Xmid = nullptr, *H2 = nullptr, *st2 = nullptr, *U = nullptr, *A = nullptr;
    };
    std::vector<VitTensor> vtens;
    int vNP = 0, vT = 0, vD = 0, vM = 0, vPK = 0;
    float *vP = nullptr, *vE = nullptr, *vX0 = nullptr, *vXout = nullptr, *vHc = nullptr, *vstf = nullptr;
    float *vdX = nullptr, *vdH = nullptr, *vdQKV = nullptr, *vdO = nullptr, *vdU = nullptr, *vdyxh = nullptr,
          *vdE = nullptr, *vdHc = nullptr;
    std::vector<VitAct> vl;
    // BF16 mode: bf16 GEMM operands and the tcgen05 descriptors of every projection
    struct VitB {
        __nv_bfloat16 *H1 = nullptr, *O = nullptr, *H2 = nullptr, *A = nullptr;
    };
    struct VitMaps {
        CUtensorMap fwd, dg, wg_g, wg_x, fwd128, dg128;
    };
    std::vector<VitB> vlb;
    std::vector<VitMaps> vmaps;  // [0] patch, [1 + 4l + {0 qkv, 1 proj, 2 fc1, 3 fc2}], [last] head
    // vdXb / vdXb1: fc2's gradient operand of even / odd layers (layer l's LayerNorm-1 backward
    // writes layer l−1's while layer l's weight gradients still read its own)
    __nv_bfloat16 *vPb = nullptr, *vHcb = nullptr, *vdXb = nullptr, *vdXb1 = nullptr, *vdXb2 = nullptr, *vdUb = nullptr,
                  *vdQKVb = nullptr, *vdEb = nullptr, *vdzb = nullptr;
    float* vwpart = nullptr;  // row-split wgrad partials
    int64_t vwpart_cap = 0;
    std::vector<float*> vvec;  // sampled 1-D tensors [chunk][n] (LayerNorm g/b, cls, pos), else null
    std::vector<CUtensorMap> cmap_hf, cmap_hd;  // conv3 HALO: 1-row (W + 2)-pixel boxes of the input / dY
    std::vector<char> halo_fwd, halo_dgrad;
    float* bias_rows_scr = nullptr;  // chunk sums of many bias partials (launch_bias_grad_rows)
    int64_t bias_rows_cap = 0;
    std::vector<char> wcps;  // conv2 weight gradient: CTAs per SM (1 or 2)
    std::vector<char> wgrad_eps;  // ε-fused, sample-accumulating weight gradient (no per-sample partials)
    StemRowMaps cmap_stem;      // the stem input: 1 … 8-row boxes of padded rows, 8 channels, no swizzle
    int stem_layer = -1;       // the layer on stem_fwd_kernel (-1: none)
    std::vector<Conv64RowMaps> rowmaps;  // conv64 weight gradient: multi-row TMA boxes
    std::vector<char> conv64;  // stage-1 64 → 64 layers on the W-stationary tap-paired kernel (both passes)
    __nv_bfloat16* fcG = nullptr;   // FC output gradient, [S][B][round8(O)]
    // TMA descriptors (BF16)
    std::vector<CUtensorMap> map_fwdB, map_dgradB, map_wgG, map_wgX;
    int map_B = 0;  // the B_loc the BF16 descriptors are encoded for
    // bookkeeping
    std::string err;
    int64_t launches = 0;
    bool prof = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_next = 0;
    std::vector<std::string> prof_names;
    std::vector<double> prof_ms;
    std::vector<int64_t> prof_n;
    std::vector<void*> allocs;

    int set_err(int code, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        g_last_error = buf;
        return code;
    }
    template <class T>
    bool alloc(T** p, size_t n) {
        void* q = nullptr;
        if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return false;
        cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T));
        allocs.push_back(q);
        *p = reinterpret_cast<T*>(q);
        return true;
    }
    int prof_class(const char* name) {
        for (size_t i = 0; i < prof_names.size(); ++i)
            if (prof_names[i] == name) return (int)i;
        prof_names.push_back(name);
        prof_ms.push_back(0.0);
        prof_n.push_back(0);
        return (int)prof_names.size() - 1;
    }
    void prof_flush() {
        if (pending.empty()) return;
        cudaStreamSynchronize(st);
        for (auto& p : pending) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.second.first, p.second.second);
            prof_ms[p.first] += ms;
            prof_n[p.first] += 1;
        }
        pending.clear();
        ev_next = 0;
    }
    static bool skip_class(const char* cls) {
        static const char* e = getenv("BNN_EXP_SKIP");
        return e && strstr(e, cls) != nullptr;
    }
    template <class F>
    void launch(const char* cls, F&& f, int kernels = 1) {
        if (skip_class(cls)) return;  // timing experiments only (BNN_EXP_SKIP=class[,class]): wrong results
        int c = -1;
        cudaEvent_t a = nullptr, b = nullptr;
        if (prof) {
            c = prof_class(cls);
            if (ev_next + 2 > ev_pool.size()) prof_flush();
            if (ev_next + 2 > ev_pool.size()) {
                for (int i = 0; i < 256; ++i) {
                    cudaEvent_t e;
                    cudaEventCreate(&e);
                    ev_pool.push_back(e);
                }
            }
            a = ev_pool[ev_next++];
            b = ev_pool[ev_next++];
            cudaEventRecord(a, st);
        }
        if constexpr (std::is_same_v<decltype(f()), int>)
            launches += f();  // the launcher reports how many kernels it launched
        else {
            f();
            launches += kernels;
        }
        if (prof) {
            cudaEventRecord(b, st);
            pending.push_back({c, {a, b}});
        }
    }
};

// NVTX range of one host-side phase (header-only NVTX v3: a no-op unless a tool such as
// nsys / ncu --nvtx is attached). Names: bnn.step, bnn.partial, bnn.chunk, bnn.forward,
// bnn.backward, bnn.exchange, bnn.finalize, bnn.predict.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Side-stream fork/join: work enqueued on the returned stream after fork_side() runs
// concurrently with what follows on c->st until join_side(). While profiling, everything
// stays on c->st (class timing needs a single stream).
inline cudaStream_t fork_side(bnn_ctx* c) {
    if (c->prof || !c->side) return c->st;
    cudaEventRecord(c->ev_fork, c->st);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    return c->side;
}
inline void join_side(bnn_ctx* c) {
    if (c->prof || !c->side) return;
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(c->st, c->ev_join, 0);
    if (c->side2) {
        cudaEventRecord(c->ev_join2, c->side2);
        cudaStreamWaitEvent(c->st, c->ev_join2, 0);
    }
    if (c->side3) {
        cudaEventRecord(c->ev_join3, c->side3);
        cudaStreamWaitEvent(c->st, c->ev_join3, 0);
    }
}
inline cudaStream_t fork_side2(bnn_ctx* c) {
    if (c->prof || !c->side2) return c->st;
    cudaEventRecord(c->ev_fork2, c->st);
    cudaStreamWaitEvent(c->side2, c->ev_fork2, 0);
    return c->side2;
}

// Chunk phases (exact aggregation):
//   kPhaseFull    forward, per-sample loss head, backward (Alg. 1 l.7-12 for the chunk)
//   kPhaseStats   forward + the mean-prediction statistic only
//   kPhaseMeanBwd (forward unless skip_fwd,) mean-prediction loss head from gstats, backward
enum { kPhaseFull = 0, kPhaseStats = 1, kPhaseMeanBwd = 2 };

// gradient exchange (comm.cu)
int comm_init(bnn_ctx* c, const uint8_t* uid, int world, int rank);
int comm_check(bnn_ctx* c, ncclResult_t r, const char* what);
int comm_sync(bnn_ctx* c, cudaStream_t st);
void comm_destroy(bnn_ctx* c);
void ar_begin(bnn_ctx* c);
int ar_layer_done(bnn_ctx* c, int l, cudaStream_t w0, cudaStream_t w1);
int ar_finish(bnn_ctx* c, cudaStream_t st);

// ViT entry points (runtime_vit.cu)
int build_vit(bnn_ctx* c);
int alloc_vit(bnn_ctx* c);
int vit_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, int B, int B_glob, int S_glob,
              int Sc, uint32_t s0, uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss);
int vit_chunk_bf16(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, int B, int B_glob, int S_glob,
                   int Sc, uint32_t s0, uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss);

// ResNet entry points (runtime_resnet.cu)
int alloc_resnet_bf16(bnn_ctx* c);
int resnet_bf16_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls,
                      const float* yreg, int B, int B_glob, int S_glob, int Sc, uint32_t s0,
                      uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss,
                      int phase = kPhaseFull, bool skip_fwd = false, const float* gstats = nullptr);
void resnet_bf16_forward(bnn_ctx* c, const float* mu, const float* x, int Sc, int B,
                         uint64_t seed, uint32_t step, uint32_t s0, bool aug);
SampledLayer sampled(const bnn_ctx* c, int l, const float* mu);

#define CUDA_TRY(ctx, expr)                                                                  \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return (ctx)->set_err(BNN_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));    \
    } while (0)

#define NCCL_TRY(ctx, expr)                                                                  \
    do {                                                                                     \
        ncclResult_t r_ = (expr);                                                            \
        if (r_ != ncclSuccess)                                                               \
            return (ctx)->set_err(BNN_ERR_COMM, "%s: %s", #expr, ncclGetErrorString(r_));    \
    } while (0)

