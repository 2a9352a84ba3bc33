// runtime.cu — the step orchestrator and the C ABI (L4) of libbnn.so.
//
// One bnn_ctx per rank/GPU. bnn_init builds the layer graph and parameter layout, allocates
// every workspace buffer, encodes the TMA descriptors of the BF16 path and creates the NCCL
// communicator. bnn_elbo_step then only enqueues kernels on the context stream (no
// allocation, no host synchronisation unless the loss is requested on the host):
//   K7 σ prologue → per sample chunk: sampled forward (K2 / K11), loss head (K6), sampled
//   dgrad (K4 / K11), wgrad with sample accumulation (K5 / K11), bias grads → one NCCL
//   SUM-allreduce of [acc_μ | acc_ρ | L_data] → K8 finalize + KL.
// Sample sharding, data sharding and the K×G hybrid grid only
// change which global samples (EPS-v1 keys) and which examples a rank processes; the
// global 1/(S·B) pre-scaling makes the flat allreduce sum compose over both axes
// (reading R8).
#include "ctx.cuh"

namespace bnn_rt {
thread_local std::string g_last_error;
}

namespace {

int build_layers(bnn_ctx* c) {
    const bnn_model_desc& m = c->model;
    int64_t off = 0;
    auto add = [&](int cin, int cout, int k, int stride, int pad) {
        LayerDesc L{cin, cout, k, stride, pad, 0, 0, 0, 0};
        L.t_w = (uint32_t)(2 * c->layers.size());
        L.t_b = L.t_w + 1;
        L.off_w = off;
        off += (int64_t)cout * k * k * cin;
        L.off_b = off;
        off += cout;
        c->layers.push_back(L);
    };
    if (m.kind == BNN_MODEL_MLP) {
        if (m.n_widths < 2 || m.n_widths > 16)
            return c->set_err(BNN_ERR_CONFIG, "MLP needs 2 <= n_widths <= 16");
        for (int i = 0; i < m.n_widths; ++i) {
            if (m.widths[i] <= 0) return c->set_err(BNN_ERR_CONFIG, "MLP widths must be > 0");
            c->widths.push_back(m.widths[i]);
        }
        for (int i = 1; i < m.n_widths; ++i) add(m.widths[i - 1], m.widths[i], 1, 1, 0);
        c->O = m.widths[m.n_widths - 1];
    } else if (m.kind == BNN_MODEL_RESNET18) {
        // CIFAR ResNet-18 without BatchNorm (R12); tensor order: stem, then per block
        // conv1, conv2, [1×1 projection], then the linear head.
        if (m.in_h < 4 || m.in_w < 4 || m.in_c < 1 || m.n_classes < 1)
            return c->set_err(BNN_ERR_CONFIG, "ResNet needs in_h, in_w >= 4, in_c, n_classes >= 1");
        const int bw = m.base_width > 0 ? m.base_width : 64;
        add(m.in_c, bw, 3, 1, 1);
        int width = bw;
        for (int stage = 0; stage < 4; ++stage) {
            const int cout = bw << stage;
            for (int blk = 0; blk < 2; ++blk) {
                const int stride = (stage > 0 && blk == 0) ? 2 : 1;
                add(width, cout, 3, stride, 1);
                add(cout, cout, 3, 1, 1);
                if (stride != 1 || width != cout) add(width, cout, 1, stride, 0);
                width = cout;
            }
        }
        add(width, m.n_classes, 1, 1, 0);
        c->O = m.n_classes;
    } else if (m.kind == BNN_MODEL_VIT) {
        return build_vit(c);  // its own tensor table (runtime_vit.cu)
    } else {
        return c->set_err(BNN_ERR_CONFIG, "unknown model kind %d", m.kind);
    }
    c->P = off;
    c->P_pad = round_up(off, 64);
    c->acc_total = 2 * c->P_pad + 64;
    if (2 * c->layers.size() >= 4095) return c->set_err(BNN_ERR_CONFIG, "too many tensors (t < 4095)");
    return BNN_OK;
}

}  // namespace
SampledLayer sampled(const bnn_ctx* c, int l, const float* mu) {
    const LayerDesc& L = c->layers[l];
    SampledLayer s;
    s.mu = mu;
    s.sigma = c->sigma;
    s.off_w = L.off_w;
    s.off_b = L.off_b;
    s.N = L.cout;
    s.K = L.cin * L.k * L.k;
    s.t_w = L.t_w;
    s.t_b = L.t_b;
    return s;
}

namespace {

// TMA descriptors of the BF16 MLP path for a batch of B rows per sample. The kernels store
// activations and gradients with sample stride B·ld (the step's B_loc), so the descriptors are
// re-encoded whenever a step's B_loc differs from the last one (host-side encode, no launch);
// TMA zero-fills rows ≥ B, which the wgrad reduction over batch rows relies on.
int mlp_encode_maps(bnn_ctx* c, int B) {
    const int L = (int)c->layers.size();
    const int Sc = c->chunk;
    c->map_fwdB.resize(L);
    c->map_dgradB.resize(L);
    c->map_wgG.resize(L);
    c->map_wgX.resize(L);
    for (int l = 0; l < L; ++l) {
        const void* in = l == 0 ? c->xb : c->act[l];
        const int depth = l == 0 ? 1 : Sc;
        if (!make_map(&c->map_fwdB[l], in, c->widths[l], B, depth, c->ld[l], 256) ||
            !make_map(&c->map_wgX[l], in, c->widths[l], B, depth, c->ld[l], 64) ||
            !make_map(&c->map_dgradB[l], c->grad[l], c->widths[l + 1], B, Sc, c->ld[l + 1], 256) ||
            !make_map(&c->map_wgG[l], c->grad[l], c->widths[l + 1], B, Sc, c->ld[l + 1], 64))
            return c->set_err(BNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (layer %d)", l);
    }
    c->map_B = B;
    return BNN_OK;
}

int alloc_mlp(bnn_ctx* c) {
    const int L = (int)c->layers.size();
    const int B = c->B_max, Sc = c->chunk;
    const size_t es = c->bf16 ? 2 : 4;
    c->ld.resize(L + 1);
    for (int l = 0; l <= L; ++l) c->ld[l] = c->bf16 ? (int)round_up(c->widths[l], 8) : c->widths[l];
    c->act.assign(L, nullptr);
    for (int l = 1; l < L; ++l) {
        void* p;
        if (cudaMalloc(&p, (size_t)Sc * B * c->ld[l] * es) != cudaSuccess)
            return c->set_err(BNN_ERR_CUDA, "out of memory (activations)");
        cudaMemset(p, 0, (size_t)Sc * B * c->ld[l] * es);
        c->allocs.push_back(p);
        c->act[l] = p;
    }
    c->grad.assign(L, nullptr);
    for (int l = 0; l < L; ++l) {
        void* p;
        const size_t n = (size_t)Sc * B * c->ld[l + 1] * es;
        if (cudaMalloc(&p, n) != cudaSuccess) return c->set_err(BNN_ERR_CUDA, "out of memory (grads)");
        cudaMemset(p, 0, n);
        c->allocs.push_back(p);
        c->grad[l] = p;
    }
    if (!c->alloc(&c->logits, (size_t)Sc * B * c->O) || !c->alloc(&c->lossrow, (size_t)Sc * B))
        return c->set_err(BNN_ERR_CUDA, "out of memory (logits)");
    int sumN = 0;  // the grouped bias launch keeps every layer's [2][S][N_l] block
    for (int l = 0; l < L; ++l) sumN += c->widths[l + 1];
    if (!c->alloc(&c->db_scratch, (size_t)2 * Sc * sumN)) return c->set_err(BNN_ERR_CUDA, "out of memory");
    if (c->bf16) {
        if (!c->alloc(&c->dz_f32, (size_t)Sc * B * c->O)) return c->set_err(BNN_ERR_CUDA, "out of memory");
        c->dbpart.assign(L, nullptr);
        const int nbc = (B + 15) / 16;
        for (int l = 0; l + 1 < L; ++l)
            if (!c->alloc(&c->dbpart[l], (size_t)Sc * nbc * c->widths[l + 1]))
                return c->set_err(BNN_ERR_CUDA, "out of memory");
    }
    if (c->bf16) {
        __nv_bfloat16* xb;
        if (!c->alloc(&xb, (size_t)B * c->ld[0])) return c->set_err(BNN_ERR_CUDA, "out of memory");
        c->xb = xb;
        return mlp_encode_maps(c, B);
    }
    return BNN_OK;
}

// ------------------------------------------------------------------ one chunk of samples
// phases: kPhaseFull / kPhaseStats / kPhaseMeanBwd (ctx.cuh)
int mlp_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls,
              const float* yreg, int B, int B_glob, int S_glob, int Sc, uint32_t s0,
              uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss,
              int phase = kPhaseFull, bool skip_fwd = false, const float* gstats = nullptr) {
    NvtxRange nvtx_("bnn.chunk");
    const int L = (int)c->layers.size();
    cudaStream_t st = c->st;
    SampleKeys kk{make_key(seed), step, s0};
    const float scale = c->model.loss == BNN_LOSS_CE ? 1.0f / ((float)S_glob * B_glob)
                                                     : 1.0f / ((float)S_glob * B_glob * c->O);
    if (!c->bf16) {
        // ---------------- FP32 SIMT path (parity mode)
        for (int l = 0; l < L && !skip_fwd; ++l) {
            SampledLayer sl = sampled(c, l, mu);
            const float* A = l == 0 ? x : (const float*)c->act[l];
            const int64_t sA = l == 0 ? 0 : (int64_t)B * c->ld[l];
            float* Z = l == L - 1 ? c->logits : (float*)c->act[l + 1];
            const int64_t sZ = (int64_t)B * (l == L - 1 ? c->O : c->ld[l + 1]);
            const DropArgs dr = c->drop_for(l, l < L - 1, B);
            c->launch("fwd", [&] { launch_fwd_fp32(sl, kk, dr, Sc, B, A, sA, Z, sZ, l < L - 1, st); });
        }
        if (phase == kPhaseStats) {
            c->launch("loss", [&] { launch_mean_stats(c->logits, Sc, B, c->O, c->mkind(), ycls, c->mstats, (int)(s0 - (uint32_t)(c->kidx * (S_glob / c->K))), st); });
            return BNN_OK;
        }
        if (phase == kPhaseMeanBwd)
            c->launch("loss", [&] {
                launch_mean_loss_head(c->logits, Sc, B, c->O, c->mkind(), ycls, yreg, gstats, S_glob,
                                      c->grad[L - 1], c->O, false, nullptr, st);
            });
        else
            c->launch("loss", [&] {
                launch_loss_head(c->logits, Sc, B, c->O, c->model.loss, ycls, yreg, c->grad[L - 1], c->O,
                                 false, c->lossrow, nullptr, st);
            });
        for (int l = L - 1; l >= 0; --l) {
            SampledLayer sl = sampled(c, l, mu);
            const float* Gl = (const float*)c->grad[l];
            const int64_t sG = (int64_t)B * c->ld[l + 1];
            const float* A = l == 0 ? x : (const float*)c->act[l];
            const int64_t sA = l == 0 ? 0 : (int64_t)B * c->ld[l];
            c->launch("wgrad", [&] {
                launch_wgrad_fp32(sl, kk, Sc, B, Gl, sG, A, sA, scale, acc_mu, acc_rho, st);
            });
            c->launch("bias", [&] {
                return launch_bias_grad(sl, kk, Sc, Gl, B, c->ld[l + 1], sG, scale, c->db_scratch, acc_mu,
                                 acc_rho, st);
            });
            if (l > 0)
                c->launch("dgrad", [&] {
                    launch_dgrad_fp32(sl, kk, c->drop_for(l - 1, true, B), Sc, B, Gl, sG, (const float*)c->act[l], sA,
                                      (float*)c->grad[l - 1], (int64_t)B * c->ld[l], st);
                });
        }
    } else {
        // ---------------- BF16 tcgen05 path
        if (B > 256 * 64) return c->set_err(BNN_ERR_CONFIG, "B_loc too large");
        const int nb = (int)round_up(std::min(B, 256), 16);
        for (int l = 0; l < L && !skip_fwd; ++l) {
            TcGenArgs a{};
            a.L = sampled(c, l, mu);
            a.kk = kk;
            a.mode = 0;
            a.B = B;
            a.b_shared = l == 0 ? 1 : 0;
            a.M = a.L.N;
            a.R = a.L.K;
            a.nb = nb;
            a.out_f32 = l == L - 1;
            a.relu = l < L - 1;
            a.out = l == L - 1 ? (void*)c->logits : c->act[l + 1];
            a.ldo = l == L - 1 ? c->O : c->ld[l + 1];
            a.out_stride_s = (int64_t)B * a.ldo;
            a.vec_ok = (a.L.K % 4 == 0 && a.L.off_w % 4 == 0) ? 1 : 0;
            a.drop = c->drop_for(l, l < L - 1, B);
            a.mu_only = c->mcd;
            c->launch("fwd", [&] { launch_gen_gemm(c->map_fwdB[l], a, Sc, st); });
        }
        if (phase == kPhaseStats) {
            c->launch("loss", [&] { launch_mean_stats(c->logits, Sc, B, c->O, c->mkind(), ycls, c->mstats, (int)(s0 - (uint32_t)(c->kidx * (S_glob / c->K))), st); });
            return BNN_OK;
        }
        if (phase == kPhaseMeanBwd)
            c->launch("loss", [&] {
                launch_mean_loss_head(c->logits, Sc, B, c->O, c->mkind(), ycls, yreg, gstats, S_glob,
                                      c->grad[L - 1], c->ld[L], true, c->dz_f32, st);
            });
        else
            c->launch("loss", [&] {
                launch_loss_head(c->logits, Sc, B, c->O, c->model.loss, ycls, yreg, c->grad[L - 1],
                                 c->ld[L], true, c->lossrow, c->dz_f32, st);
            });
        bool forked = false;
        if (phase == kPhaseFull) {  // the loss reduction overlaps the backward
            cudaStream_t ss = fork_side(c);
            forked = true;
            c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, ss); });
        }
        for (int l = L - 1; l >= 1; --l) {
            TcGenArgs a{};
            a.L = sampled(c, l, mu);
            a.kk = kk;
            a.mode = 1;
            a.B = B;
            a.b_shared = 0;
            a.M = a.L.K;
            a.R = a.L.N;
            a.nb = nb;
            a.out = c->grad[l - 1];
            a.ldo = c->ld[l];
            a.out_stride_s = (int64_t)B * c->ld[l];
            a.mask = (const __nv_bfloat16*)c->act[l];
            a.ldm = c->ld[l];
            a.mask_stride_s = (int64_t)B * c->ld[l];
            a.vec_ok = (a.L.K % 4 == 0 && a.L.off_w % 4 == 0) ? 1 : 0;
            a.dbpart = c->dbpart[l - 1];
            a.dbpart_stride_s = (int64_t)((B + 15) / 16) * a.L.K;
            a.drop = c->drop_for(l - 1, true, B);
            a.mu_only = c->mcd;
            c->launch("dgrad", [&] { launch_gen_gemm(c->map_dgradB[l], a, Sc, st); });
        }
        for (int l0 = 0; l0 < L; l0 += kMaxBiasGroup) {
            BiasGroup bg{};
            for (int l = l0; l < std::min(L, l0 + kMaxBiasGroup); ++l) {
                const bool last = l == L - 1;
                const int nbc = (B + 15) / 16;
                const int i = bg.n++;
                bg.L[i] = sampled(c, l, mu);
                bg.parts[i] = last ? c->dz_f32 : c->dbpart[l];
                bg.nparts[i] = last ? B : nbc;
                bg.ldp[i] = last ? c->O : bg.L[i].N;
                bg.strideS[i] = (int64_t)bg.nparts[i] * bg.ldp[i];
            }
            // the bias gradients (dgrad's fp32 partials, the loss head's seed) overlap the
            // wgrad GEMM, which leaves SMs free (128 tiles on 148 SMs)
            cudaStream_t ss = fork_side(c);
            forked = true;
            c->launch("bias", [&] {
                launch_bias_grad_grouped(bg, kk, Sc, scale, c->db_scratch, acc_mu, acc_rho, ss);
            }, 2);
        }
        for (int l0 = 0; l0 < L; l0 += kMaxWgradLayers) {
            TcWgradMaps maps;
            TcWgradArgs w{};
            w.skip_eps = c->mcd;
            w.kk = kk;
            w.S = Sc;
            w.B = B;
            w.scale = scale;
            w.acc_mu = acc_mu;
            w.acc_rho = acc_rho;
            int base = 0;
            for (int l = l0; l < std::min(L, l0 + kMaxWgradLayers); ++l) {
                WgradLayer& wl = w.lay[w.nlayers];
                wl.L = sampled(c, l, mu);
                wl.mtiles = (wl.L.N + 127) / 128;
                wl.ktiles = (wl.L.K + kWgradTileK - 1) / kWgradTileK;
                wl.tile_base = base;
                wl.b_shared = l == 0 ? 1 : 0;
                base += wl.mtiles * wl.ktiles;
                maps.g[w.nlayers] = c->map_wgG[l];
                maps.x[w.nlayers] = c->map_wgX[l];
                ++w.nlayers;
            }
            c->launch("wgrad", [&] { launch_wgrad_tc(maps, w, st); });
        }
        if (forked) join_side(c);
        if (phase == kPhaseFull) return BNN_OK;  // loss reduced on the side stream
    }
    if (phase == kPhaseFull)
        c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, st); });
    return BNN_OK;
}


// ------------------------------------------------------------------ ResNet graph (C3–C5)
int conv_out_dim(int x, int k, int st, int p) { return (x + 2 * p - k) / st + 1; }

int alloc_resnet(bnn_ctx* c) {
    const bnn_model_desc& m = c->model;
    auto buf = [&](int H, int W, int C) {
        c->rbufs.push_back(RBuf{H, W, C, nullptr, nullptr});
        return (int)c->rbufs.size() - 1;
    };
    auto conv = [&](int src, int li, int res, int relu) {
        const LayerDesc& L = c->layers[li];
        const RBuf& S = c->rbufs[src];
        const int d = buf(conv_out_dim(S.H, L.k, L.stride, L.pad), conv_out_dim(S.W, L.k, L.stride, L.pad),
                          L.cout);
        c->rops.push_back(ROp{0, li, src, d, res, relu});
        return d;
    };
    int l = 0;
    int cur = buf(m.in_h, m.in_w, m.in_c);
    cur = conv(cur, l++, -1, 1);  // stem
    int width = c->layers[0].cout;
    for (int stage = 0; stage < 4; ++stage) {
        const int cout = c->layers[0].cout << stage;
        for (int blk = 0; blk < 2; ++blk) {
            const int stride = (stage > 0 && blk == 0) ? 2 : 1;
            const bool proj = stride != 1 || width != cout;
            const int l1 = l++, l2 = l++, lp = proj ? l++ : -1;
            const int in = cur;
            const int a = conv(in, l1, -1, 1);
            const int sc = proj ? conv(in, lp, -1, 0) : in;
            cur = conv(a, l2, sc, 1);
            width = cout;
        }
    }
    const int g = buf(1, 1, width);
    c->rops.push_back(ROp{1, -1, cur, g, -1, 0});
    c->rlogits = conv(g, l++, -1, 0);
    if (c->bf16) return alloc_resnet_bf16(c);
    const int B = c->B_max, Sc = c->chunk;
    for (size_t i = 0; i < c->rbufs.size(); ++i) {
        RBuf& b = c->rbufs[i];
        const size_t n = (size_t)Sc * B * b.H * b.W * b.C;
        if (!c->alloc(&b.val, n) || !c->alloc(&b.grad, i == 0 ? 1 : n))
            return c->set_err(BNN_ERR_CUDA, "out of memory (ResNet activations)");
    }
    int maxN = 0;
    for (auto& L : c->layers) maxN = std::max(maxN, L.cout);
    if (!c->alloc(&c->db_scratch, (size_t)2 * Sc * maxN) || !c->alloc(&c->lossrow, (size_t)Sc * B))
        return c->set_err(BNN_ERR_CUDA, "out of memory");
    return BNN_OK;
}

ConvShape shape_of(const bnn_ctx* c, const ROp& op, int B) {
    const LayerDesc& L = c->layers[op.layer];
    const RBuf& S = c->rbufs[op.src];
    const RBuf& D = c->rbufs[op.dst];
    return ConvShape{B, S.H, S.W, S.C, D.H, D.W, D.C, L.k, L.stride, L.pad};
}
int64_t per_sample(const RBuf& b, int B) { return (int64_t)B * b.H * b.W * b.C; }

// forward of one chunk; X0/sX0 = (augmented) input and its per-sample stride
void resnet_forward(bnn_ctx* c, const float* mu, const SampleKeys& kk, int Sc, int B, const float* X0,
                    int64_t sX0) {
    cudaStream_t st = c->st;
    auto val = [&](int i) -> const float* { return i == 0 ? X0 : c->rbufs[i].val; };
    auto sval = [&](int i) -> int64_t { return i == 0 ? sX0 : per_sample(c->rbufs[i], B); };
    for (const ROp& op : c->rops) {
        if (op.type == 1) {
            const RBuf& S = c->rbufs[op.src];
            c->launch("gap", [&] { launch_gap_fwd(c->rbufs[op.src].val, Sc * B, S.H * S.W, S.C, c->rbufs[op.dst].val, st); });
            continue;
        }
        SampledLayer sl = sampled(c, op.layer, mu);
        ConvShape cs = shape_of(c, op, B);
        const float* R = op.res >= 0 ? val(op.res) : nullptr;
        const int64_t sR = op.res >= 0 ? sval(op.res) : 0;
        c->launch("fwd", [&] {
            launch_conv_fwd_fp32(sl, kk, Sc, cs, val(op.src), sval(op.src), R, sR, c->rbufs[op.dst].val,
                                 per_sample(c->rbufs[op.dst], B), op.relu != 0, st);
        });
    }
}

int resnet_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, const float* yreg,
                 int B, int B_glob, int S_glob, int Sc, uint32_t s0, uint64_t seed, uint32_t step,
                 float* acc_mu, float* acc_rho, float* acc_loss, int phase = kPhaseFull,
                 bool skip_fwd = false, const float* gstats = nullptr) {
    cudaStream_t st = c->st;
    SampleKeys kk{make_key(seed), step, s0};
    const float scale = c->model.loss == BNN_LOSS_CE ? 1.0f / ((float)S_glob * B_glob)
                                                     : 1.0f / ((float)S_glob * B_glob * c->O);
    const RBuf& in = c->rbufs[0];
    const float* X0 = x;
    int64_t sX0 = 0;
    if (c->cfg.aug == BNN_AUG_PER_SAMPLE) {
        if (!skip_fwd)
            c->launch("aug", [&] {
                launch_augment(x, Sc, B, in.H, in.W, in.C, seed, step, s0, c->gidx * B, c->rbufs[0].val, st);
            });
        X0 = c->rbufs[0].val;
        sX0 = per_sample(in, B);
    }
    if (!skip_fwd) resnet_forward(c, mu, kk, Sc, B, X0, sX0);
    RBuf& lg = c->rbufs[c->rlogits];
    if (phase == kPhaseStats) {
        c->launch("loss", [&] { launch_mean_stats(lg.val, Sc, B, c->O, c->mkind(), ycls, c->mstats, (int)(s0 - (uint32_t)(c->kidx * (S_glob / c->K))), st); });
        return BNN_OK;
    }
    if (phase == kPhaseMeanBwd)
        c->launch("loss", [&] {
            launch_mean_loss_head(lg.val, Sc, B, c->O, c->mkind(), ycls, yreg, gstats, S_glob, lg.grad, c->O,
                                  false, nullptr, st);
        });
    else
        c->launch("loss", [&] {
            launch_loss_head(lg.val, Sc, B, c->O, c->model.loss, ycls, yreg, lg.grad, c->O, false, c->lossrow,
                             nullptr, st);
        });
    std::vector<char> written(c->rbufs.size(), 0);
    written[c->rlogits] = 1;
    auto val = [&](int i) -> const float* { return i == 0 ? X0 : c->rbufs[i].val; };
    auto sval = [&](int i) -> int64_t { return i == 0 ? sX0 : per_sample(c->rbufs[i], B); };
    for (int oi = (int)c->rops.size() - 1; oi >= 0; --oi) {
        const ROp& op = c->rops[oi];
        RBuf& D = c->rbufs[op.dst];
        if (op.type == 1) {
            const RBuf& S = c->rbufs[op.src];
            c->launch("gap", [&] { launch_gap_bwd(D.grad, Sc * B, S.H * S.W, S.C, c->rbufs[op.src].grad, st); });
            written[op.src] = 1;
            continue;
        }
        const int64_t nD = Sc * per_sample(D, B);
        if (op.relu) c->launch("mask", [&] { launch_relu_mask(D.grad, D.val, nD, st); });
        SampledLayer sl = sampled(c, op.layer, mu);
        ConvShape cs = shape_of(c, op, B);
        const int64_t sD = per_sample(D, B);
        c->launch("wgrad", [&] {
            launch_conv_wgrad_fp32(sl, kk, Sc, cs, D.grad, sD, val(op.src), sval(op.src), scale, acc_mu, acc_rho, st);
        });
        c->launch("bias", [&] {
            return launch_bias_grad(sl, kk, Sc, D.grad, B * D.H * D.W, D.C, sD, scale, c->db_scratch, acc_mu, acc_rho, st);
        });
        if (op.res >= 0) {
            RBuf& Rb = c->rbufs[op.res];
            if (written[op.res])
                c->launch("add", [&] { launch_add(Rb.grad, D.grad, nD, st); });
            else
                CUDA_TRY(c, cudaMemcpyAsync(Rb.grad, D.grad, sizeof(float) * nD, cudaMemcpyDeviceToDevice, st));
            written[op.res] = 1;
        }
        if (op.src != 0) {
            RBuf& Sb = c->rbufs[op.src];
            const bool acc = written[op.src] != 0;
            c->launch("dgrad", [&] {
                launch_conv_dgrad_fp32(sl, kk, Sc, cs, D.grad, sD, Sb.grad, per_sample(Sb, B), acc, st);
            });
            written[op.src] = 1;
        }
    }
    if (phase == kPhaseFull)
        c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, st); });
    return BNN_OK;
}

int check_step_args(bnn_ctx* c, int B_loc, int B_glob, int S_glob) {
    if (B_loc <= 0 || B_loc > c->B_max)
        return c->set_err(BNN_ERR_CONFIG, "0 < B_loc <= max_B_loc (%d) violated: B_loc=%d", c->B_max, B_loc);
    if (B_glob != B_loc * c->G)
        return c->set_err(BNN_ERR_CONFIG, "B_global == G * B_loc violated (%d != %d * %d)", B_glob, c->G, B_loc);
    if (S_glob <= 0 || S_glob % c->K != 0)
        return c->set_err(BNN_ERR_CONFIG, "S mod K == 0 violated (S=%d, K=%d)", S_glob, c->K);
    if (S_glob / c->K > c->S_loc_max)
        return c->set_err(BNN_ERR_CONFIG, "S/K <= max_S_loc violated (%d > %d)", S_glob / c->K, c->S_loc_max);
    if (S_glob >= (1 << 20)) return c->set_err(BNN_ERR_CONFIG, "S < 2^20 (EPS-v1 counter) violated");
    if (c->bf16 && B_loc != c->map_B) {
        // the BF16 ResNet's descriptors, scratch splits and per-layer grids are laid out for
        // max_B_loc in bnn_init; the MLP's descriptors are re-encoded for the new batch size
        if (c->model.kind != BNN_MODEL_MLP)
            return c->set_err(BNN_ERR_CONFIG,
                              "BF16 ResNet: B_loc == max_B_loc required (B_loc=%d, max_B_loc=%d); "
                              "create a context with max_B_loc = B_loc for a smaller batch", B_loc, c->B_max);
        // the previous step's kernels read the old descriptors by value (kernel parameters),
        // so re-encoding on the host does not race with work still in flight
        int rc = mlp_encode_maps(c, B_loc);
        if (rc) return rc;
    }
    return BNN_OK;
}

int any_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, const float* yreg, int B,
              int B_glob, int S_glob, int Sc, uint32_t s0, uint64_t seed, uint32_t step, float* am, float* ar,
              float* al, int phase, bool skip_fwd, const float* gstats) {
    if (c->model.kind == BNN_MODEL_MLP)
        return mlp_chunk(c, mu, x, ycls, yreg, B, B_glob, S_glob, Sc, s0, seed, step, am, ar, al, phase, skip_fwd,
                         gstats);
    if (c->bf16)
        return resnet_bf16_chunk(c, mu, x, ycls, yreg, B, B_glob, S_glob, Sc, s0, seed, step, am, ar, al, phase,
                                 skip_fwd, gstats);
    return resnet_chunk(c, mu, x, ycls, yreg, B, B_glob, S_glob, Sc, s0, seed, step, am, ar, al, phase, skip_fwd,
                        gstats);
}

// local partial sums into acc (zeroed first).
// Exact aggregation (c->agg): stats_out != NULL → only this rank's statistic
// (bnn_mean_stats); gstats_in != NULL → the backward with the caller's merged statistic
// (bnn_elbo_partial_mean); neither → both phases with the statistic exchanged over the
// communicator (one allgather between forward and backward) or, for world 1, used as is.
int run_partial(bnn_ctx* c, const float* mu, const float* rho, const float* x, const int32_t* ycls,
                const float* yreg, int B_loc, int B_glob, int S_glob, uint64_t seed, uint32_t step,
                float* acc, const float* gstats_in = nullptr, float* stats_out = nullptr) {
    NvtxRange nvtx_("bnn.partial");
    int rc = check_step_args(c, B_loc, B_glob, S_glob);
    if (rc) return rc;
    if (c->model.loss == BNN_LOSS_CE && !ycls) return c->set_err(BNN_ERR_CONFIG, "CE loss needs int32 labels");
    if (c->model.loss == BNN_LOSS_MSE && !yreg) return c->set_err(BNN_ERR_CONFIG, "MSE loss needs fp32 targets");
    if ((gstats_in || stats_out) && !c->agg)
        return c->set_err(BNN_ERR_CONFIG, "mean statistics need a BNN_LOSS_*_MEAN model");
    cudaStream_t st = c->st;
    // the bf16 cast of the input overlaps the σ prologue (side stream, joined before the chunks)
    const bool cast = c->bf16 && c->model.kind == BNN_MODEL_MLP;
    if (cast) {
        cudaStream_t ss = fork_side(c);
        const int K0 = c->widths[0];
        c->launch("cast", [&] { launch_to_bf16(x, B_loc, K0, c->ld[0], c->xb, ss); });
    }
    if (!stats_out) CUDA_TRY(c, cudaMemsetAsync(acc, 0, sizeof(float) * c->acc_total, st));
    if (c->mcd)  // MC dropout: the weights are μ (σ = 0 ⇒ W_s = fma(0, ε, μ) = μ), R25
        CUDA_TRY(c, cudaMemsetAsync(c->sigma, 0, sizeof(float) * c->P, st));
    else
        c->launch("sigma", [&] { launch_sigma(rho, c->sigma, c->P, st); });
    if (cast) join_side(c);
    const int S_loc = S_glob / c->K;
    float* accm = acc;
    float* accr = acc ? acc + c->P_pad : nullptr;
    float* accl = acc ? acc + 2 * c->P_pad : nullptr;
    if (c->agg) {
        const bool single = S_loc <= c->chunk;  // activations of the stats pass stay valid
        const float* gstats = gstats_in;
        if (!gstats_in) {
            CUDA_TRY(c, cudaMemsetAsync(c->mstats, 0, sizeof(float) * (size_t)B_loc * c->stat_w, st));
            for (int s = 0; s < S_loc; s += c->chunk) {
                const int Sc = std::min(c->chunk, S_loc - s);
                const uint32_t s0 = (uint32_t)(c->kidx * S_loc + s);
                rc = any_chunk(c, mu, x, ycls, yreg, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr,
                               accl, kPhaseStats, false, nullptr);
                if (rc) return rc;
            }
            if (stats_out) {
                CUDA_TRY(c, cudaMemcpyAsync(stats_out, c->mstats, sizeof(float) * (size_t)B_loc * c->stat_w,
                                            cudaMemcpyDeviceToDevice, st));
                CUDA_TRY(c, cudaGetLastError());
                return BNN_OK;
            }
            if (c->comm) {
                // Σ over the K sample groups of this data group, in rank order (PAPER.md:281
                // "additional communication"); one allgather, then a deterministic merge
                const int64_t n = (int64_t)B_loc * c->stat_w;
                rc = comm_check(c, ncclAllGather(c->mstats, c->mgather, (size_t)n, ncclFloat32, c->comm, st),
                                "ncclAllGather(mean statistic)");
                if (rc) return rc;
                c->launch("loss", [&] { launch_mean_merge(c->mgather, c->cfg.world, c->G, c->gidx, n, c->mstats_g, c->gnll ? c->O : 0, S_loc, st); });
                gstats = c->mstats_g;
            } else {
                if (c->K != 1)
                    return c->set_err(BNN_ERR_CONFIG, "K > 1 without a communicator: use bnn_mean_stats + bnn_elbo_partial_mean");
                gstats = c->mstats;
            }
        }
        for (int s = 0; s < S_loc; s += c->chunk) {
            const int Sc = std::min(c->chunk, S_loc - s);
            const uint32_t s0 = (uint32_t)(c->kidx * S_loc + s);
            c->ar_live = c->ar_enabled && s + Sc >= S_loc;  // acc segments final in the last chunk
            c->ar_live_used |= c->ar_live;
            rc = any_chunk(c, mu, x, ycls, yreg, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr, accl,
                           kPhaseMeanBwd, single && !gstats_in, gstats);
            c->ar_live = false;
            if (rc) return rc;
        }
        if (c->kidx == 0) {  // the data loss counts each example once: sample group 0 adds it
            const float sc = c->model.loss == BNN_LOSS_CE ? 1.0f / (float)B_glob : 1.0f / ((float)B_glob * c->O);
            c->launch("loss", [&] {
                launch_mean_loss_value(gstats, B_loc, c->O, c->mkind(), yreg, S_glob, sc, accl, st);
            });
        }
        CUDA_TRY(c, cudaGetLastError());
        return BNN_OK;
    }
    for (int s = 0; s < S_loc; s += c->chunk) {
        const int Sc = std::min(c->chunk, S_loc - s);
        const uint32_t s0 = (uint32_t)(c->kidx * S_loc + s);
        c->ar_live = c->ar_enabled && s + Sc >= S_loc;  // acc segments final in the last chunk
        c->ar_live_used |= c->ar_live;
        if (c->model.kind == BNN_MODEL_VIT)
            rc = vit_chunk(c, mu, x, ycls, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr, accl);
        else if (c->model.kind == BNN_MODEL_MLP)
            rc = mlp_chunk(c, mu, x, ycls, yreg, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr, accl);
        else if (c->bf16)
            rc = resnet_bf16_chunk(c, mu, x, ycls, yreg, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr, accl);
        else
            rc = resnet_chunk(c, mu, x, ycls, yreg, B_loc, B_glob, S_glob, Sc, s0, seed, step, accm, accr, accl);
        c->ar_live = false;
        if (rc) return rc;
    }
    CUDA_TRY(c, cudaGetLastError());
    return BNN_OK;
}

int run_finalize(bnn_ctx* c, const float* mu, const float* rho, const float* acc, float* loss_dev,
                 float* gmu, float* grho) {
    NvtxRange nvtx_("bnn.finalize");
    cudaStream_t st = c->st;
    c->launch("finalize", [&] {
        launch_finalize(c->mcd, mu, rho, acc, acc + c->P_pad, acc + 2 * c->P_pad, c->P, c->cfg.dataset_size,
                        gmu, grho, c->kl_part, c->n_part, c->lossbuf, st);
    }, 2);
    if (loss_dev) CUDA_TRY(c, cudaMemcpyAsync(loss_dev, c->lossbuf, sizeof(float), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaGetLastError());
    return BNN_OK;
}

int read_loss(bnn_ctx* c, double* loss_host) {
    float h = 0.f;
    CUDA_TRY(c, cudaMemcpyAsync(&h, c->lossbuf, sizeof(float), cudaMemcpyDeviceToHost, c->st));
    int rc = comm_sync(c, c->st);  // polls the communicator: a dead peer is BNN_ERR_COMM, not a hang
    if (rc) return rc;
    *loss_host = h;
    if (!std::isfinite(h)) return c->set_err(BNN_ERR_NUMERIC, "non-finite loss %f", (double)h);
    return BNN_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int bnn_get_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_last_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
        return BNN_ERR_COMM;
    }
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return BNN_OK;
}

int bnn_init(const bnn_model_desc* model, const bnn_config* cfg, bnn_ctx** out) {
    if (!model || !cfg || !out) {
        g_last_error = "null argument";
        return BNN_ERR_CONFIG;
    }
    *out = nullptr;
    bnn_ctx* c = new bnn_ctx();
    c->model = *model;
    c->cfg = *cfg;
    auto fail = [&](int rc) {
        bnn_destroy(c);
        return rc;
    };
    // ---- config invariants
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return fail(c->set_err(BNN_ERR_CONFIG, "0 <= rank < world violated"));
    if (cfg->mode == BNN_MODE_SAMPLE_SHARDED) {
        c->K = cfg->world;
        c->G = 1;
    } else if (cfg->mode == BNN_MODE_DATA_SHARDED) {
        c->K = 1;
        c->G = cfg->world;
    } else if (cfg->mode == BNN_MODE_HYBRID) {
        c->K = cfg->K;
        c->G = cfg->G;
        if (c->K < 1 || c->G < 1 || c->K * c->G != cfg->world)
            return fail(c->set_err(BNN_ERR_CONFIG, "world == K*G violated (%d != %d*%d)", cfg->world, cfg->K, cfg->G));
    } else {
        return fail(c->set_err(BNN_ERR_CONFIG, "unknown mode %d", cfg->mode));
    }
    c->kidx = cfg->rank / c->G;
    c->gidx = cfg->rank % c->G;
    if (cfg->max_B_loc <= 0 || cfg->max_S_loc <= 0)
        return fail(c->set_err(BNN_ERR_CONFIG, "max_B_loc > 0 and max_S_loc > 0 required"));
    if (!(cfg->dataset_size > 0)) return fail(c->set_err(BNN_ERR_CONFIG, "dataset_size > 0 required"));
    if (cfg->precision != BNN_PREC_FP32 && cfg->precision != BNN_PREC_BF16)
        return fail(c->set_err(BNN_ERR_CONFIG, "unknown precision"));
    if (cfg->aug != BNN_AUG_NONE && cfg->aug != BNN_AUG_PER_SAMPLE)
        return fail(c->set_err(BNN_ERR_CONFIG, "unknown aug mode"));
    if (model->loss < BNN_LOSS_CE || model->loss > BNN_LOSS_GNLL_MEAN)
        return fail(c->set_err(BNN_ERR_CONFIG, "unknown loss"));
    if (model->loss >= BNN_LOSS_CE_MEAN) {
        // exact aggregation: the base loss family, plus the mean-statistic exchange
        c->agg = 1;
        c->gnll = model->loss == BNN_LOSS_GNLL_MEAN ? 1 : 0;
        if (c->gnll && model->kind != BNN_MODEL_MLP)
            return fail(c->set_err(BNN_ERR_CONFIG, "the Gaussian NLL loss is implemented for MLP models"));
        // bf16 rounding of the predictions perturbs the S-sample variance that the seeds divide
        // by (1/v, 1/v²): measured 5-7 % gradient error, beyond the BF16 bar (R24)
        if (c->gnll && cfg->precision != BNN_PREC_FP32)
            return fail(c->set_err(BNN_ERR_CONFIG, "the Gaussian NLL loss needs precision FP32"));
        c->model.loss = model->loss == BNN_LOSS_CE_MEAN ? BNN_LOSS_CE : BNN_LOSS_MSE;
    }
    if (model->method != BNN_METHOD_VI && model->method != BNN_METHOD_MCD)
        return fail(c->set_err(BNN_ERR_CONFIG, "unknown method"));
    if (model->method == BNN_METHOD_MCD) {  // MC dropout (R25)
        if (model->kind != BNN_MODEL_MLP) return fail(c->set_err(BNN_ERR_CONFIG, "MC dropout is implemented for MLP models"));
        if (!(model->dropout_p >= 0.0f && model->dropout_p < 1.0f))
            return fail(c->set_err(BNN_ERR_CONFIG, "0 <= dropout_p < 1 violated"));
        c->mcd = 1;
        c->p24 = (uint32_t)llround((double)model->dropout_p * 16777216.0);
        c->inv_keep = (float)(1.0 / (1.0 - (double)model->dropout_p));
    }
    c->bf16 = cfg->precision == BNN_PREC_BF16;
    c->B_max = cfg->max_B_loc;
    c->S_loc_max = cfg->max_S_loc;
    c->chunk = cfg->sample_chunk > 0 ? std::min(cfg->sample_chunk, cfg->max_S_loc) : cfg->max_S_loc;
    int rc = build_layers(c);
    if (rc) return fail(rc);
    if (model->kind == BNN_MODEL_MLP && cfg->aug != BNN_AUG_NONE)
        return fail(c->set_err(BNN_ERR_CONFIG, "augmentation applies to image models only"));
    c->in_elems = model->kind == BNN_MODEL_MLP ? (int64_t)model->widths[0]
                                              : (int64_t)model->in_h * model->in_w * model->in_c;
    // ---- device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(c->set_err(BNN_ERR_CUDA, "no CUDA device (there is no CPU fallback)"));
    if (cfg->device < 0 || cfg->device >= ndev) return fail(c->set_err(BNN_ERR_CONFIG, "bad device ordinal"));
    if (cudaSetDevice(cfg->device) != cudaSuccess) return fail(c->set_err(BNN_ERR_CUDA, "cudaSetDevice failed"));
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, cfg->device);
    if (prop.major != 10)
        return fail(c->set_err(BNN_ERR_CUDA, "device is sm_%d%d; libbnn is built for sm_100a only", prop.major, prop.minor));
    c->st = reinterpret_cast<cudaStream_t>(cfg->stream);  // NULL = legacy default stream
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join2, cudaEventDisableTiming) != cudaSuccess)
        return fail(c->set_err(BNN_ERR_CUDA, "stream/event creation failed"));
    // ---- workspace
    c->n_part = finalize_partials_count(c->P);
    if (!c->alloc(&c->sigma, c->P) || !c->alloc(&c->acc, c->acc_total) ||
        !c->alloc(&c->kl_part, c->n_part) || !c->alloc(&c->lossbuf, 4) ||
        !c->alloc(&c->x_stage, (size_t)c->B_max * c->in_elems) ||
        !c->alloc(&c->ycls_stage, c->B_max) || !c->alloc(&c->yreg_stage, (size_t)c->B_max * c->O) ||
        !c->alloc(&c->p_mean, (size_t)c->B_max * c->G * c->O) || !c->alloc(&c->p_m2, (size_t)c->B_max * c->G * c->O) ||
        !c->alloc(&c->g_means, (size_t)c->B_max * c->G * c->O * cfg->world) ||
        !c->alloc(&c->g_m2s, (size_t)c->B_max * c->G * c->O * cfg->world) ||
        !c->alloc(&c->g_counts, cfg->world))
        return fail(c->set_err(BNN_ERR_CUDA, "out of device memory"));
    rc = model->kind == BNN_MODEL_MLP ? alloc_mlp(c) : model->kind == BNN_MODEL_VIT ? alloc_vit(c) : alloc_resnet(c);
    if (rc) return fail(rc);
    if (c->agg) {
        c->stat_w = c->gnll ? 2 * c->O : c->model.loss == BNN_LOSS_CE ? 1 : c->O;
        const size_t n = (size_t)c->B_max * c->stat_w;
        if (!c->alloc(&c->mstats, n) || !c->alloc(&c->mstats_g, n) || !c->alloc(&c->mgather, n * cfg->world))
            return fail(c->set_err(BNN_ERR_CUDA, "out of device memory"));
    }
    // ---- communicator
    if (cfg->nccl_uid) {  // also for world == 1 (exercises the NCCL path on one GPU)
        if (cfg->comm_timeout_ms > 0) c->comm_timeout_ms = cfg->comm_timeout_ms;
        else if (const char* e = getenv("BNN_COMM_TIMEOUT_MS")) c->comm_timeout_ms = atof(e);
        rc = comm_init(c, cfg->nccl_uid, cfg->world, cfg->rank);
        if (rc) return fail(rc);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(c->set_err(BNN_ERR_CUDA, "init sync failed"));
    *out = c;
    return BNN_OK;
}

int bnn_param_layout(bnn_ctx* c, int64_t* n_params, int32_t* n_tensors, bnn_tensor_info* infos,
                     int32_t max_infos) {
    if (!c) return BNN_ERR_CONFIG;
    if (n_params) *n_params = c->P;
    if (c->model.kind == BNN_MODEL_VIT) {
        const int nt = (int)c->vtens.size();
        if (n_tensors) *n_tensors = nt;
        for (int t = 0; infos && t < nt && t < max_infos; ++t) {
            infos[t].t = t;
            infos[t].offset = c->vtens[t].off;
            infos[t].rows = c->vtens[t].rows;
            infos[t].cols = c->vtens[t].cols;
            infos[t].is_bias = c->vtens[t].rows == 1 ? 1 : 0;
        }
        return BNN_OK;
    }
    const int nt = (int)c->layers.size() * 2;
    if (n_tensors) *n_tensors = nt;
    if (infos) {
        for (int t = 0; t < nt && t < max_infos; ++t) {
            const LayerDesc& L = c->layers[t / 2];
            bnn_tensor_info& I = infos[t];
            I.t = t;
            I.is_bias = t % 2;
            if (t % 2 == 0) {
                I.offset = L.off_w;
                I.rows = L.cout;
                I.cols = L.k * L.k * L.cin;
            } else {
                I.offset = L.off_b;
                I.rows = 1;
                I.cols = L.cout;
            }
        }
    }
    return BNN_OK;
}

int bnn_acc_layout(bnn_ctx* c, int64_t* rho_offset, int64_t* loss_offset, int64_t* total) {
    if (!c) return BNN_ERR_CONFIG;
    if (rho_offset) *rho_offset = c->P_pad;
    if (loss_offset) *loss_offset = 2 * c->P_pad;
    if (total) *total = c->acc_total;
    return BNN_OK;
}

int bnn_elbo_partial(bnn_ctx* c, const float* mu, const float* rho, const float* x, const int32_t* ycls,
                     const float* yreg, int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                     uint32_t step, float* acc_dev) {
    if (!c || !mu || !rho || !x || !acc_dev) return BNN_ERR_CONFIG;
    return run_partial(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step, acc_dev);
}

int bnn_mean_stats(bnn_ctx* c, const float* mu, const float* rho, const float* x, const int32_t* ycls,
                   int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed, uint32_t step,
                   float* stats_dev) {
    if (!c || !mu || !rho || !x || !stats_dev) return BNN_ERR_CONFIG;
    if (!c->agg) return c->set_err(BNN_ERR_CONFIG, "bnn_mean_stats needs a BNN_LOSS_*_MEAN model");
    // MSE statistics need no targets; pass a dummy non-null pointer through the label checks
    const float* yreg = c->model.loss == BNN_LOSS_MSE ? x : nullptr;
    return run_partial(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step, nullptr, nullptr,
                       stats_dev);
}

int bnn_elbo_partial_mean(bnn_ctx* c, const float* mu, const float* rho, const float* x,
                          const int32_t* ycls, const float* yreg, int32_t B_loc, int32_t B_global,
                          int32_t S_global, uint64_t seed, uint32_t step, const float* stats_global_dev,
                          float* acc_dev) {
    if (!c || !mu || !rho || !x || !acc_dev || !stats_global_dev) return BNN_ERR_CONFIG;
    return run_partial(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step, acc_dev,
                       stats_global_dev);
}

int bnn_mean_merge(bnn_ctx* c, const float* stats_all, int32_t n_groups, int32_t B_loc, int32_t S_global,
                   float* out) {
    if (!c || !stats_all || !out || n_groups <= 0 || B_loc <= 0) return BNN_ERR_CONFIG;
    if (!c->agg) return c->set_err(BNN_ERR_CONFIG, "bnn_mean_merge needs a BNN_LOSS_*_MEAN model");
    if (S_global % n_groups != 0) return c->set_err(BNN_ERR_CONFIG, "S mod n_groups == 0 violated");
    const int64_t n = (int64_t)B_loc * c->stat_w;
    c->launch("loss", [&] {
        launch_mean_merge(stats_all, n_groups, 1, 0, n, out, c->gnll ? c->O : 0, S_global / n_groups, c->st);
    });
    CUDA_TRY(c, cudaGetLastError());
    return BNN_OK;
}

int bnn_finalize(bnn_ctx* c, const float* mu, const float* rho, const float* acc_dev, float* loss_dev,
                 float* gmu, float* grho) {
    if (!c || !mu || !rho || !acc_dev || !gmu || !grho) return BNN_ERR_CONFIG;
    return run_finalize(c, mu, rho, acc_dev, loss_dev, gmu, grho);
}

namespace {
// This rank's partial + the one SUM-allreduce of [acc_μ | acc_ρ | L_data] (PAPER.md:243,
// :263-264); afterwards c->acc holds the global sums on every rank.
int run_reduced(bnn_ctx* c, const float* mu, const float* rho, const float* x, const int32_t* ycls,
                const float* yreg, int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                uint32_t step) {
    if (c->cfg.world > 1 && !c->comm)
        return c->set_err(BNN_ERR_CONFIG, "world > 1 without a communicator: use bnn_elbo_partial + bnn_finalize");
    if (c->comm) {
        // bucketed exchange: the ResNet backward reduces each finished bucket of layers on the
        // comm stream (ar_layer_done); the tail and L_data follow (ar_finish)
        ar_begin(c);
        c->ar_enabled = c->model.kind != BNN_MODEL_MLP && c->bf16;
    }
    int rc = run_partial(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step, c->acc);
    c->ar_enabled = false;
    if (rc) return rc;
    if (c->comm) {
        int cls = -1;
        cudaEvent_t a = nullptr, b = nullptr;
        if (c->prof) {
            cls = c->prof_class("allreduce");
            if (c->ev_next + 2 > c->ev_pool.size()) c->prof_flush();
            if (c->ev_next + 2 > c->ev_pool.size())
                for (int i = 0; i < 64; ++i) {
                    cudaEvent_t e;
                    cudaEventCreate(&e);
                    c->ev_pool.push_back(e);
                }
            a = c->ev_pool[c->ev_next++];
            b = c->ev_pool[c->ev_next++];
            cudaEventRecord(a, c->st);
        }
        NvtxRange nv("bnn.exchange");
        rc = ar_finish(c, c->st);
        c->ar_live_used = false;
        if (rc) return rc;
        if (c->prof) {
            cudaEventRecord(b, c->st);
            c->pending.push_back({cls, {a, b}});
        }
    }
    return BNN_OK;
}

int check_adam(bnn_ctx* c, const bnn_adam* h, AdamHyper* out) {
    if (!h) return c->set_err(BNN_ERR_CONFIG, "null bnn_adam");
    if (!(h->lr >= 0.f) || !(h->beta1 >= 0.f && h->beta1 < 1.f) || !(h->beta2 >= 0.f && h->beta2 < 1.f) ||
        !(h->eps > 0.f) || h->t < 1)
        return c->set_err(BNN_ERR_CONFIG, "Adam hyper-parameters: lr >= 0, 0 <= beta < 1, eps > 0, t >= 1 violated");
    out->lr = h->lr;
    out->beta1 = h->beta1;
    out->beta2 = h->beta2;
    out->eps = h->eps;
    out->omb1 = (float)(1.0 - (double)h->beta1);
    out->omb2 = (float)(1.0 - (double)h->beta2);
    out->bc1 = (float)(1.0 - std::pow((double)h->beta1, (double)h->t));
    out->bc2 = (float)(1.0 - std::pow((double)h->beta2, (double)h->t));
    return BNN_OK;
}

int run_finalize_adam(bnn_ctx* c, float* mu, float* rho, const float* acc, const bnn_adam* hp,
                      float* m_mu, float* v_mu, float* m_rho, float* v_rho, float* loss_dev,
                      float* gmu, float* grho) {
    NvtxRange nvtx_("bnn.finalize");
    if (c->mcd) return c->set_err(BNN_ERR_CONFIG, "the fused Adam step is for BNN_METHOD_VI models");
    AdamHyper h;
    int rc = check_adam(c, hp, &h);
    if (rc) return rc;
    if (!m_mu || !v_mu || !m_rho || !v_rho) return c->set_err(BNN_ERR_CONFIG, "null Adam moment buffer");
    cudaStream_t st = c->st;
    c->launch("finalize", [&] {
        launch_finalize_adam(mu, rho, acc, acc + c->P_pad, acc + 2 * c->P_pad, c->P, c->cfg.dataset_size, h,
                             m_mu, v_mu, m_rho, v_rho, gmu, grho, c->kl_part, c->n_part, c->lossbuf, st);
    }, 2);
    if (loss_dev) CUDA_TRY(c, cudaMemcpyAsync(loss_dev, c->lossbuf, sizeof(float), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaGetLastError());
    return BNN_OK;
}
}  // namespace

int bnn_elbo_step(bnn_ctx* c, const float* mu, const float* rho, const float* x, const int32_t* ycls,
                  const float* yreg, int32_t B_loc, int32_t B_global, int32_t S_global, uint64_t seed,
                  uint32_t step, float* loss_dev, double* loss_host, float* gmu, float* grho) {
    NvtxRange nvtx_("bnn.step");
    if (!c || !mu || !rho || !x || !gmu || !grho) {
        if (c) return c->set_err(BNN_ERR_CONFIG, "null tensor argument");
        return BNN_ERR_CONFIG;
    }
    int rc = run_reduced(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step);
    if (rc) return rc;
    rc = run_finalize(c, mu, rho, c->acc, loss_dev, gmu, grho);
    if (rc) return rc;
    if (loss_host) return read_loss(c, loss_host);
    return BNN_OK;
}

int bnn_finalize_adam(bnn_ctx* c, float* mu, float* rho, const float* acc_dev, const bnn_adam* h,
                      float* m_mu, float* v_mu, float* m_rho, float* v_rho, float* loss_dev,
                      float* gmu, float* grho) {
    if (!c || !mu || !rho || !acc_dev) return BNN_ERR_CONFIG;
    return run_finalize_adam(c, mu, rho, acc_dev, h, m_mu, v_mu, m_rho, v_rho, loss_dev, gmu, grho);
}

int bnn_elbo_step_adam(bnn_ctx* c, float* mu, float* rho, const float* x, const int32_t* ycls,
                       const float* yreg, int32_t B_loc, int32_t B_global, int32_t S_global,
                       uint64_t seed, uint32_t step, const bnn_adam* h, float* m_mu, float* v_mu,
                       float* m_rho, float* v_rho, float* loss_dev, double* loss_host, float* gmu,
                       float* grho) {
    if (!c || !mu || !rho || !x) {
        if (c) return c->set_err(BNN_ERR_CONFIG, "null tensor argument");
        return BNN_ERR_CONFIG;
    }
    int rc = run_reduced(c, mu, rho, x, ycls, yreg, B_loc, B_global, S_global, seed, step);
    if (rc) return rc;
    rc = run_finalize_adam(c, mu, rho, c->acc, h, m_mu, v_mu, m_rho, v_rho, loss_dev, gmu, grho);
    if (rc) return rc;
    if (loss_host) return read_loss(c, loss_host);
    return BNN_OK;
}

int bnn_elbo_step_host(bnn_ctx* c, const float* mu, const float* rho, const float* x_host,
                       const int32_t* ycls_host, const float* yreg_host, int32_t B_loc, int32_t B_global,
                       int32_t S_global, uint64_t seed, uint32_t step, double* loss_host, float* gmu,
                       float* grho) {
    if (!c || !x_host || !loss_host) return BNN_ERR_CONFIG;
    if (B_loc <= 0 || B_loc > c->B_max) return c->set_err(BNN_ERR_CONFIG, "0 < B_loc <= max_B_loc violated");
    const size_t in = (size_t)c->in_elems;
    CUDA_TRY(c, cudaMemcpyAsync(c->x_stage, x_host, sizeof(float) * in * B_loc, cudaMemcpyHostToDevice, c->st));
    if (ycls_host)
        CUDA_TRY(c, cudaMemcpyAsync(c->ycls_stage, ycls_host, sizeof(int32_t) * B_loc, cudaMemcpyHostToDevice, c->st));
    if (yreg_host)
        CUDA_TRY(c, cudaMemcpyAsync(c->yreg_stage, yreg_host, sizeof(float) * B_loc * c->O, cudaMemcpyHostToDevice, c->st));
    return bnn_elbo_step(c, mu, rho, c->x_stage, ycls_host ? c->ycls_stage : nullptr,
                         yreg_host ? c->yreg_stage : nullptr, B_loc, B_global, S_global, seed, step, nullptr,
                         loss_host, gmu, grho);
}

int bnn_predict(bnn_ctx* c, const float* mu, const float* rho, const float* x, int32_t B, int32_t S_global,
                uint64_t seed, uint32_t step, float* mean, float* var) {
    NvtxRange nvtx_("bnn.predict");
    if (!c || !mu || !rho || !x || !mean || !var) return BNN_ERR_CONFIG;
    if (c->G != 1) return c->set_err(BNN_ERR_CONFIG, "predict is sample-sharded only (G == 1)");
    if (c->model.kind == BNN_MODEL_VIT) return c->set_err(BNN_ERR_CONFIG, "predict: MLP and ResNet models");
    int rc = check_step_args(c, B, B * c->G, S_global);
    if (rc) return rc;
    cudaStream_t st = c->st;
    const int L = (int)c->layers.size();
    const int S_loc = S_global / c->K;
    const int BO = B * c->O;
    if (c->mcd)  // MC dropout: the weights are μ (σ = 0 ⇒ W_s = fma(0, ε, μ) = μ), R25
        CUDA_TRY(c, cudaMemsetAsync(c->sigma, 0, sizeof(float) * c->P, st));
    else
        c->launch("sigma", [&] { launch_sigma(rho, c->sigma, c->P, st); });
    if (c->bf16 && c->model.kind == BNN_MODEL_MLP)
        c->launch("cast", [&] { launch_to_bf16(x, B, c->widths[0], c->ld[0], c->xb, st); });
    // per chunk forward; stats over all local samples need all logits, so chunk == S_loc here
    if (S_loc > c->chunk) return c->set_err(BNN_ERR_CONFIG, "predict needs S/K <= sample_chunk");
    SampleKeys kk{make_key(seed), step, (uint32_t)(c->kidx * S_loc)};
    const bool is_mlp = c->model.kind == BNN_MODEL_MLP;
    if (!is_mlp && !c->bf16) resnet_forward(c, mu, kk, S_loc, B, x, 0);
    if (!is_mlp && c->bf16) resnet_bf16_forward(c, mu, x, S_loc, B, seed, step, kk.s0, false);
    const int nb = (int)round_up(std::min(B, 256), 16);
    for (int l = 0; is_mlp && l < L; ++l) {
        if (!c->bf16) {
            SampledLayer sl = sampled(c, l, mu);
            const float* A = l == 0 ? x : (const float*)c->act[l];
            const int64_t sA = l == 0 ? 0 : (int64_t)B * c->ld[l];
            float* Z = l == L - 1 ? c->logits : (float*)c->act[l + 1];
            const int64_t sZ = (int64_t)B * (l == L - 1 ? c->O : c->ld[l + 1]);
            const DropArgs dr = c->drop_for(l, l < L - 1, B);
            c->launch("fwd", [&] { launch_fwd_fp32(sl, kk, dr, S_loc, B, A, sA, Z, sZ, l < L - 1, st); });
        } else {
            TcGenArgs a{};
            a.L = sampled(c, l, mu);
            a.kk = kk;
            a.mode = 0;
            a.B = B;
            a.b_shared = l == 0 ? 1 : 0;
            a.M = a.L.N;
            a.R = a.L.K;
            a.nb = nb;
            a.out_f32 = l == L - 1;
            a.relu = l < L - 1;
            a.out = l == L - 1 ? (void*)c->logits : c->act[l + 1];
            a.ldo = l == L - 1 ? c->O : c->ld[l + 1];
            a.out_stride_s = (int64_t)B * a.ldo;
            a.vec_ok = (a.L.K % 4 == 0 && a.L.off_w % 4 == 0) ? 1 : 0;
            a.drop = c->drop_for(l, l < L - 1, B);
            a.mu_only = c->mcd;
            c->launch("fwd", [&] { launch_gen_gemm(c->map_fwdB[l], a, S_loc, st); });
        }
    }
    const float* logits = (is_mlp || c->bf16) ? c->logits : c->rbufs[c->rlogits].val;
    c->launch("predict", [&] { launch_predict_stats(logits, S_loc, B, c->O, c->model.loss, c->p_mean, c->p_m2, st); });
    const int R = c->cfg.world;
    if (c->comm && R > 1) {
        if ((rc = comm_check(c, ncclGroupStart(), "ncclGroupStart")) ||
            (rc = comm_check(c, ncclAllGather(c->p_mean, c->g_means, BO, ncclFloat32, c->comm, st), "ncclAllGather(mean)")) ||
            (rc = comm_check(c, ncclAllGather(c->p_m2, c->g_m2s, BO, ncclFloat32, c->comm, st), "ncclAllGather(M2)")) ||
            (rc = comm_check(c, ncclGroupEnd(), "ncclGroupEnd")))
            return rc;
    } else if (R > 1) {
        return c->set_err(BNN_ERR_CONFIG, "predict with world > 1 needs a communicator");
    } else {
        CUDA_TRY(c, cudaMemcpyAsync(c->g_means, c->p_mean, sizeof(float) * BO, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(c, cudaMemcpyAsync(c->g_m2s, c->p_m2, sizeof(float) * BO, cudaMemcpyDeviceToDevice, st));
    }
    std::vector<float> counts(R, (float)S_loc);
    CUDA_TRY(c, cudaMemcpyAsync(c->g_counts, counts.data(), sizeof(float) * R, cudaMemcpyHostToDevice, st));
    c->launch("predict", [&] { launch_predict_merge(c->g_means, c->g_m2s, c->g_counts, R, BO, mean, var, st); });
    CUDA_TRY(c, cudaStreamSynchronize(st));  // counts host buffer lifetime
    CUDA_TRY(c, cudaGetLastError());
    return BNN_OK;
}

int bnn_eps_fill(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r0, uint32_t nr,
                 uint32_t c0, uint32_t nc, float* out, void* stream) {
    if (!out) return BNN_ERR_CONFIG;
    launch_eps_fill(seed, step, s, t, r0, nr, c0, nc, out, reinterpret_cast<cudaStream_t>(stream));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = cudaGetErrorString(e);
        return BNN_ERR_CUDA;
    }
    return BNN_OK;
}

int bnn_eps_transform_table(int32_t which, float* out, void* stream) {
    if (!out || which < 0 || which > 2) return BNN_ERR_CONFIG;
    launch_eps_table(which, out, reinterpret_cast<cudaStream_t>(stream));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = cudaGetErrorString(e);
        return BNN_ERR_CUDA;
    }
    return BNN_OK;
}

int bnn_eps_bench(uint64_t n4, uint64_t seed, float* sink, int32_t grid, void* stream) {
    if (!sink || grid <= 0) return BNN_ERR_CONFIG;
    launch_eps_bench(n4, seed, sink, grid, reinterpret_cast<cudaStream_t>(stream));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = cudaGetErrorString(e);
        return BNN_ERR_CUDA;
    }
    return BNN_OK;
}

int bnn_profile_enable(bnn_ctx* c, int32_t on) {
    if (!c) return BNN_ERR_CONFIG;
    if (!on) c->prof_flush();
    c->prof = on != 0;
    if (on) {
        for (size_t i = 0; i < c->prof_ms.size(); ++i) {
            c->prof_ms[i] = 0.0;
            c->prof_n[i] = 0;
        }
    }
    return BNN_OK;
}

int bnn_profile_read(bnn_ctx* c, char* names, int32_t cap, double* ms, int64_t* launches, int32_t max_entries,
                     int32_t* n_entries) {
    if (!c) return BNN_ERR_CONFIG;
    c->prof_flush();
    std::string all;
    const int n = (int)std::min<size_t>(c->prof_names.size(), (size_t)max_entries);
    for (int i = 0; i < n; ++i) {
        if (i) all += ",";
        all += c->prof_names[i];
        if (ms) ms[i] = c->prof_ms[i];
        if (launches) launches[i] = c->prof_n[i];
    }
    if (names && cap > 0) {
        strncpy(names, all.c_str(), cap - 1);
        names[cap - 1] = 0;
    }
    if (n_entries) *n_entries = n;
    return BNN_OK;
}

int64_t bnn_launch_count(bnn_ctx* c) { return c ? c->launches : -1; }

int bnn_debug_layer_output(bnn_ctx* c, int32_t layer, int32_t which, float* out, int64_t cap,
                           int64_t* n_out) {
    if (!c || !out) return BNN_ERR_CONFIG;
    if (c->model.kind != BNN_MODEL_RESNET18) return c->set_err(BNN_ERR_CONFIG, "ResNet contexts only");
    for (const ROp& op : c->rops) {
        if (op.type != 0 || op.layer != layer) continue;
        const RBuf& D = c->rbufs[op.dst];
        const int64_t n = (int64_t)c->chunk * c->B_max * D.H * D.W * D.C;
        if (n > cap) return c->set_err(BNN_ERR_CONFIG, "debug buffer too small");
        if (n_out) *n_out = n;
        if (!c->bf16) {
            const float* src = which == 0 ? D.val : D.grad;
            CUDA_TRY(c, cudaMemcpyAsync(out, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->st));
        } else if (op.dst == c->rlogits) {
            CUDA_TRY(c, cudaMemcpyAsync(out, c->logits, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->st));
        } else {
            const __nv_bfloat16* src = which == 0 ? c->rbf[op.dst].val : c->rbf[op.dst].grad;
            launch_bf16_to_f32(src, n, out, c->st);
        }
        CUDA_TRY(c, cudaStreamSynchronize(c->st));
        return BNN_OK;
    }
    return c->set_err(BNN_ERR_CONFIG, "no such layer");
}

int32_t bnn_comm_buckets(bnn_ctx* c) { return c ? c->ar_buckets : 0; }

int bnn_sync(bnn_ctx* c) {
    if (!c) return BNN_ERR_CONFIG;
    return comm_sync(c, c->st);
}

const char* bnn_last_error(bnn_ctx* c) { return c ? c->err.c_str() : g_last_error.c_str(); }

void bnn_destroy(bnn_ctx* c) {
    if (!c) return;
    if (!c->allocs.empty()) cudaStreamSynchronize(c->st);
    comm_destroy(c);
    for (void* p : c->allocs) cudaFree(p);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (cudaStream_t q : {c->side, c->side2, c->side3})
        if (q) {
            cudaStreamSynchronize(q);
            cudaStreamDestroy(q);
        }
    for (cudaEvent_t e : {c->ev_fork2, c->ev_join2, c->ev_join3, c->ev_wg[0], c->ev_wg[1], c->ev_comb[0],
                          c->ev_comb[1]})
        if (e) cudaEventDestroy(e);
    for (auto e : c->wgen_ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
    delete c;
}

}  // extern "C"
