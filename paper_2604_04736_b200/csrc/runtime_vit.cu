// runtime_vit.cu — the Bayesian ViT step (use case 1):
// tensor table, workspace and the per-chunk forward + backward (FP32 and BF16 modes).
//
// Per sample chunk (Sc samples of the same B_loc examples; rows R = B·T tokens):
//   patches (crop/flip keyed by global (s, b)) → sampled patch projection → [cls; E] + pos
//   per encoder layer: LN1 → sampled QKV → softmax attention → sampled proj + residual →
//                      LN2 → sampled fc1 → GELU → sampled fc2 + residual
//   final LN of the cls rows → sampled head → per-sample CE (K6, shared with the MLP / CNN)
// and the backward in reverse. The sampled projections use the K2/K4/K5-family FP32 kernels
// of the MLP (W_s generated on chip from μ, σ and EPS-v1; never stored); the 1-D variational
// tensors (LayerNorm g/b, cls, pos) are drawn once per chunk into [Sc][n] buffers; every
// 1-D tensor's gradient (biases, g, b, cls, pos) goes through the bias-gradient reduction
// (Σ rows, then acc_μ += Σ_s, acc_ρ += Σ_s ε_s ⊙ ·).
#include "ctx.cuh"
#include "kernels_tc.cuh"
#include "kernels_vit.cuh"

namespace {

SampledLayer lin(const bnn_ctx* c, const float* mu, int t_w) {
    SampledLayer L{};
    L.mu = mu;
    L.sigma = c->sigma;
    L.off_w = c->vtens[t_w].off;
    L.off_b = c->vtens[t_w + 1].off;
    L.N = c->vtens[t_w].rows;
    L.K = c->vtens[t_w].cols;
    L.t_w = (uint32_t)t_w;
    L.t_b = (uint32_t)(t_w + 1);
    return L;
}

// a 1-D tensor t as the "bias" of a SampledLayer (the bias-gradient path reads off_b, t_b, N)
SampledLayer vec(const bnn_ctx* c, const float* mu, int t) {
    SampledLayer L{};
    L.mu = mu;
    L.sigma = c->sigma;
    L.off_w = c->vtens[t].off;
    L.off_b = c->vtens[t].off;
    L.N = c->vtens[t].cols;
    L.K = 0;
    L.t_w = L.t_b = (uint32_t)t;
    return L;
}

}  // namespace

int build_vit(bnn_ctx* c) {
    const bnn_model_desc& m = c->model;
    if (m.patch < 1 || m.in_h % m.patch || m.in_w % m.patch || m.dim < 32 || m.heads < 1 || m.dim % m.heads ||
        m.depth < 1 || m.depth > 64 || m.mlp < 1 || m.n_classes < 1 || m.in_c < 1 || m.dim % 4)
        return c->set_err(BNN_ERR_CONFIG,
                          "ViT: patch | in_h, in_w; dim %% heads == 0, dim %% 4 == 0, dim >= 32; 1 <= depth <= 64");
    if (m.dim / m.heads > 128) return c->set_err(BNN_ERR_CONFIG, "ViT: head dimension <= 128");
    c->vNP = (m.in_h / m.patch) * (m.in_w / m.patch);
    c->vT = 1 + c->vNP;
    if (c->vT > 68 || m.dim / m.heads > 68)
        return c->set_err(BNN_ERR_CONFIG, "ViT: at most 67 patches and head dimension <= 68 (attention tiles)");
    c->vD = m.dim;
    c->vM = m.mlp;
    c->vPK = m.patch * m.patch * m.in_c;
    const int D = c->vD, M = c->vM, T = c->vT;
    auto add = [&](int rows, int cols) { c->vtens.push_back({0, rows, cols}); };
    add(D, c->vPK); add(1, D); add(1, D); add(1, T * D);
    for (int l = 0; l < m.depth; ++l) {
        add(1, D); add(1, D); add(3 * D, D); add(1, 3 * D); add(D, D); add(1, D);
        add(1, D); add(1, D); add(M, D); add(1, M); add(D, M); add(1, D);
    }
    add(1, D); add(1, D); add(m.n_classes, D); add(1, m.n_classes);
    int64_t off = 0;
    for (auto& t : c->vtens) {
        t.off = off;
        off += (int64_t)t.rows * t.cols;
    }
    c->O = m.n_classes;
    c->P = off;
    c->P_pad = round_up(off, 64);
    c->acc_total = 2 * c->P_pad + 64;
    return BNN_OK;
}

int alloc_vit(bnn_ctx* c) {
    if (c->agg || c->mcd) return c->set_err(BNN_ERR_CONFIG, "ViT: per-sample CE, Bayes by backprop only");
    const int B = c->B_max, Sc = c->chunk, T = c->vT, D = c->vD, M = c->vM, L = c->model.depth;
    const int64_t R = (int64_t)B * T;
    const bool aug = c->cfg.aug == BNN_AUG_PER_SAMPLE;
    bool ok = c->alloc(&c->vP, (size_t)(aug ? Sc : 1) * B * c->vNP * c->vPK) &&
              c->alloc(&c->vE, (size_t)Sc * B * c->vNP * D) && c->alloc(&c->vX0, (size_t)Sc * R * D) &&
              c->alloc(&c->vXout, (size_t)Sc * R * D) && c->alloc(&c->vHc, (size_t)Sc * B * D) &&
              c->alloc(&c->vstf, (size_t)Sc * B * 2) && c->alloc(&c->logits, (size_t)Sc * B * c->O) &&
              c->alloc(&c->lossrow, (size_t)Sc * B) && c->alloc(&c->dz_f32, (size_t)Sc * B * c->O) &&
              c->alloc(&c->vdX, (size_t)Sc * R * D) && c->alloc(&c->vdH, (size_t)Sc * R * D) &&
              c->alloc(&c->vdQKV, (size_t)Sc * R * 3 * D) && c->alloc(&c->vdO, (size_t)Sc * R * D) &&
              c->alloc(&c->vdU, (size_t)Sc * R * M) && c->alloc(&c->vdyxh, (size_t)Sc * R * D) &&
              c->alloc(&c->vdE, (size_t)Sc * B * c->vNP * D) && c->alloc(&c->vdHc, (size_t)Sc * B * D);
    if (!ok) return c->set_err(BNN_ERR_CUDA, "out of memory (ViT)");
    c->vl.assign(L, bnn_ctx::VitAct{});
    for (int l = 0; l < L; ++l) {
        bnn_ctx::VitAct& a = c->vl[l];
        ok = c->alloc(&a.X, (size_t)Sc * R * D) && c->alloc(&a.H1, (size_t)Sc * R * D) &&
             c->alloc(&a.st1, (size_t)Sc * R * 2) && c->alloc(&a.QKV, (size_t)Sc * R * 3 * D) &&
             c->alloc(&a.Att, (size_t)Sc * B * c->model.heads * T * T) && c->alloc(&a.O, (size_t)Sc * R * D) &&
             c->alloc(&a.Xmid, (size_t)Sc * R * D) && c->alloc(&a.H2, (size_t)Sc * R * D) &&
             c->alloc(&a.st2, (size_t)Sc * R * 2) && c->alloc(&a.U, (size_t)Sc * R * M) &&
             c->alloc(&a.A, (size_t)Sc * R * M);
        if (!ok) return c->set_err(BNN_ERR_CUDA, "out of memory (ViT layer activations)");
    }
    // sampled 1-D tensors [Sc][n]: every tensor with rows == 1 that is not a linear bias
    c->vvec.assign(c->vtens.size(), nullptr);
    auto want = [&](int t) {
        if (t == 2 || t == 3) return true;                      // cls, pos
        const int nt = (int)c->vtens.size();
        if (t >= nt - 4) return t == nt - 4 || t == nt - 3;     // final LN g, b
        const int r = (t - 4) % 12;
        return r == 0 || r == 1 || r == 6 || r == 7;            // LN1 / LN2 g, b
    };
    for (int t = 0; t < (int)c->vtens.size(); ++t)
        if (want(t) && !c->alloc(&c->vvec[t], (size_t)Sc * c->vtens[t].cols))
            return c->set_err(BNN_ERR_CUDA, "out of memory (ViT sampled vectors)");
    c->vwpart_cap = (int64_t)4 << 20;  // row-split wgrad partials (launch_wgrad_fp32), 16 MB
    if (!c->alloc(&c->vwpart, (size_t)c->vwpart_cap)) return c->set_err(BNN_ERR_CUDA, "out of memory");
    const int maxN = std::max({M, 3 * D, T * D, c->O});
    if (!c->alloc(&c->db_scratch, (size_t)2 * Sc * maxN)) return c->set_err(BNN_ERR_CUDA, "out of memory");
    if (!c->bf16) return BNN_OK;
    // ---- BF16 mode: bf16 copies of every projection's input (kept for its weight gradient), the
    // output gradients as GEMM operands, and the descriptors (all widths are multiples of 8 except
    // the head's classes: pitch round_up(O, 8))
    const int NP = c->vNP, PK = c->vPK, ldO = (int)round_up(c->O, 8);
    if (PK % 8 != 0 || D % 8 != 0 || M % 8 != 0)
        return c->set_err(BNN_ERR_CONFIG, "ViT BF16: patch·patch·in_c, dim and mlp must be multiples of 8");
    c->vlb.assign(L, bnn_ctx::VitB{});
    for (int l = 0; l < L; ++l) {
        bnn_ctx::VitB& b = c->vlb[l];
        if (!(c->alloc(&b.H1, (size_t)Sc * R * D) && c->alloc(&b.O, (size_t)Sc * R * D) &&
              c->alloc(&b.H2, (size_t)Sc * R * D) && c->alloc(&b.A, (size_t)Sc * R * M)))
            return c->set_err(BNN_ERR_CUDA, "out of memory (ViT bf16 activations)");
    }
    ok = c->alloc(&c->vPb, (size_t)(aug ? Sc : 1) * B * NP * PK) && c->alloc(&c->vHcb, (size_t)Sc * B * D) &&
         c->alloc(&c->vdXb, (size_t)Sc * R * D) && c->alloc(&c->vdXb1, (size_t)Sc * R * D) &&
         c->alloc(&c->vdXb2, (size_t)Sc * R * D) &&
         c->alloc(&c->vdUb, (size_t)Sc * R * M) && c->alloc(&c->vdQKVb, (size_t)Sc * R * 3 * D) &&
         c->alloc(&c->vdEb, (size_t)Sc * B * NP * D) && c->alloc(&c->vdzb, (size_t)Sc * B * ldO);
    if (!ok) return c->set_err(BNN_ERR_CUDA, "out of memory (ViT bf16 gradients)");
    c->vmaps.assign(2 + 4 * L, bnn_ctx::VitMaps{});
    // (input X [.][rows][K], gradient G [.][rows][N]) of one projection
    auto maps = [&](bnn_ctx::VitMaps& m, const void* Xb, int K, int ldK, int rows, int xdepth, const void* Gb, int N,
                    int ldN) {
        return make_map(&m.fwd, Xb, K, rows, xdepth, ldK, 256) && make_map(&m.wg_x, Xb, K, rows, xdepth, ldK, 64) &&
               make_map(&m.dg, Gb, N, rows, Sc, ldN, 256) && make_map(&m.wg_g, Gb, N, rows, Sc, ldN, 64) &&
               make_map(&m.fwd128, Xb, K, rows, xdepth, ldK, 128) && make_map(&m.dg128, Gb, N, rows, Sc, ldN, 128);
    };
    ok = maps(c->vmaps[0], c->vPb, PK, PK, B * NP, aug ? Sc : 1, c->vdEb, D, D);
    for (int l = 0; l < L && ok; ++l) {
        const bnn_ctx::VitB& b = c->vlb[l];
        ok = maps(c->vmaps[1 + 4 * l], b.H1, D, D, (int)R, Sc, c->vdQKVb, 3 * D, 3 * D) &&
             maps(c->vmaps[2 + 4 * l], b.O, D, D, (int)R, Sc, c->vdXb2, D, D) &&
             maps(c->vmaps[3 + 4 * l], b.H2, D, D, (int)R, Sc, c->vdUb, M, M) &&
             maps(c->vmaps[4 + 4 * l], b.A, M, M, (int)R, Sc, (l & 1) ? c->vdXb1 : c->vdXb, D, D);
    }
    ok = ok && maps(c->vmaps[1 + 4 * L], c->vHcb, D, D, B, Sc, c->vdzb, c->O, ldO);
    if (!ok) return c->set_err(BNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (ViT)");
    c->map_B = B;
    return BNN_OK;
}

namespace {
// Z[s][rows][N] (fp32) = Xb · W_sᵀ + b_s on tcgen05, W_s generated on chip (K2, kernels_tc.cu)
void proj_fwd(bnn_ctx* c, const SampledLayer& Lw, const SampleKeys& kk, const bnn_ctx::VitMaps& m, int Sc, int rows,
              bool shared, float* Z, cudaStream_t st, const float* res = nullptr) {
    TcGenArgs a{};
    a.L = Lw;
    a.kk = kk;
    a.mode = 0;
    a.B = rows;
    a.b_shared = shared ? 1 : 0;
    a.M = Lw.N;
    a.R = Lw.K;
    a.nb = (int)round_up(std::min(rows, 256), 16);
    a.out = Z;
    a.ldo = Lw.N;
    a.out_stride_s = (int64_t)rows * Lw.N;
    a.out_f32 = 1;
    a.relu = 0;
    a.res_f32 = res;
    a.vec_ok = (Lw.K % 4 == 0 && Lw.off_w % 4 == 0) ? 1 : 0;
    c->launch("fwd", [&] { launch_gen_gemm_ws(m.fwd, m.fwd128, a, Sc, st); });
}
// dX[s][rows][K] (fp32) = G_s · W_s (K4, W_s regenerated on chip; bf16 operands, fp32 result)
void proj_dgrad(bnn_ctx* c, const SampledLayer& Lw, const SampleKeys& kk, const bnn_ctx::VitMaps& m, int Sc, int rows,
                float* dXb, cudaStream_t st) {
    TcGenArgs a{};
    a.L = Lw;
    a.kk = kk;
    a.mode = 1;
    a.B = rows;
    a.M = Lw.K;
    a.R = Lw.N;
    a.nb = (int)round_up(std::min(rows, 256), 16);
    a.out = dXb;
    a.out_f32 = 1;
    a.ldo = Lw.K;
    a.out_stride_s = (int64_t)rows * Lw.K;
    a.vec_ok = (Lw.K % 4 == 0 && Lw.off_w % 4 == 0) ? 1 : 0;
    c->launch("dgrad", [&] { launch_gen_gemm_ws(m.dg, m.dg128, a, Sc, st); });
}
// weight gradients of up to 4 projections in one K5 launch (ε-weighted sample sums in the epilogue)
struct WgItem {
    SampledLayer L;
    const bnn_ctx::VitMaps* m;
    int shared;
};
void proj_wgrad(bnn_ctx* c, const SampleKeys& kk, int Sc, int rows, float scale, float* am, float* ar,
                const WgItem* it, int n, cudaStream_t st) {
    TcWgradMaps maps;
    TcWgradArgs w{};
    w.kk = kk;
    w.S = Sc;
    w.B = rows;
    w.scale = scale;
    w.acc_mu = am;
    w.acc_rho = ar;
    int base = 0;
    for (int i = 0; i < n; ++i) {
        WgradLayer& wl = w.lay[w.nlayers];
        wl.L = it[i].L;
        wl.mtiles = (wl.L.N + 127) / 128;
        wl.ktiles = (wl.L.K + kWgradTileK - 1) / kWgradTileK;
        wl.tile_base = base;
        wl.b_shared = it[i].shared;
        base += wl.mtiles * wl.ktiles;
        maps.g[w.nlayers] = it[i].m->wg_g;
        maps.x[w.nlayers] = it[i].m->wg_x;
        ++w.nlayers;
    }
    // row splits so that up to 148 CTAs run in ONE wave (the tiles alone are 14–40; a 149th CTA
    // would be a second wave), within the scratch
    int64_t need = 0;
    for (int i = 0; i < n; ++i) need += 2 * (int64_t)it[i].L.N * it[i].L.K;
    w.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({148 /* SMs */ / base, (rows + 511) / 512,
                                                            c->vwpart_cap / std::max<int64_t>(need, 1)}));
    w.part = c->vwpart;
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
        w.part_off[i] = off;
        off += 2 * (int64_t)w.nsplit * it[i].L.N * it[i].L.K;
    }
    c->launch("wgrad", [&] { launch_wgrad_tc(maps, w, st); });
}
}  // namespace

// BF16 mode: the projections (patch, QKV, proj, fc1, fc2, head) on the tcgen05 sampled-layer
// kernels with W_s formed on chip (K2 fwd, K4 dgrad) and the ε-weighted sample sums of the
// weight gradient in the K5 epilogue; their inputs are stored once more in bf16 (GEMM operands),
// their outputs in fp32; LayerNorm, attention, GELU and the residual stream stay fp32 (R14:
// bf16 operands, fp32 accumulation).
int vit_chunk_bf16(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, int B, int B_glob, int S_glob,
                   int Sc, uint32_t s0, uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss) {
    NvtxRange nvtx_("bnn.chunk");
    cudaStream_t st = c->st;
    if (B != c->map_B)
        return c->set_err(BNN_ERR_CONFIG, "ViT BF16: B_loc == max_B_loc required (B_loc=%d, max_B_loc=%d)", B, c->B_max);
    const SampleKeys kk{make_key(seed), step, s0};
    const int T = c->vT, D = c->vD, M = c->vM, L = c->model.depth, Hh = c->model.heads, NP = c->vNP;
    const int64_t R = (int64_t)B * T, RD = R * D;
    const int nt = (int)c->vtens.size(), ldO = (int)round_up(c->O, 8);
    const float scale = 1.0f / ((float)S_glob * B_glob);
    const bool aug = c->cfg.aug == BNN_AUG_PER_SAMPLE;
    {
        NvtxRange nv("bnn.forward");
        for (int t = 0; t < nt; ++t)
            if (c->vvec[t])
                c->launch("sample", [&] {
                    launch_vit_sample_vec(mu, c->sigma, c->vtens[t].off, (uint32_t)t, c->vtens[t].cols, kk, Sc,
                                          c->vvec[t], st);
                });
        c->launch("elem", [&] {
            launch_vit_patchify(x, aug ? Sc : 1, B, c->model.in_h, c->model.in_w, c->model.in_c, c->model.patch,
                                aug ? 1 : 0, seed, step, s0, c->gidx * B, c->vPb, st);
        });
        proj_fwd(c, lin(c, mu, 0), kk, c->vmaps[0], Sc, B * NP, !aug, c->vE, st);
        // the layers' inputs are written in place: the embedding into layer 0's X, each fc2
        // (with its residual fused into the GEMM epilogue) into the next layer's X
        c->launch("elem", [&] { launch_vit_embed(c->vE, c->vvec[2], c->vvec[3], Sc, B, T, D, c->vl[0].X, st); });
        for (int l = 0; l < L; ++l) {
            bnn_ctx::VitAct& a = c->vl[l];
            bnn_ctx::VitB& b = c->vlb[l];
            const int tb = 4 + 12 * l;
            c->launch("ln", [&] {
                launch_vit_ln_fwd(a.X, Sc, (int)R, D, RD, D, c->vvec[tb], c->vvec[tb + 1], b.H1, D, RD, a.st1, st);
            });
            proj_fwd(c, lin(c, mu, tb + 2), kk, c->vmaps[1 + 4 * l], Sc, (int)R, false, a.QKV, st);
            c->launch("attn", [&] { launch_vit_attn_fwd(a.QKV, Sc, B, T, D, Hh, b.O, a.Att, st); });
            proj_fwd(c, lin(c, mu, tb + 4), kk, c->vmaps[2 + 4 * l], Sc, (int)R, false, a.Xmid, st, a.X);
            c->launch("ln", [&] {
                launch_vit_ln_fwd(a.Xmid, Sc, (int)R, D, RD, D, c->vvec[tb + 6], c->vvec[tb + 7], b.H2, D, RD, a.st2, st);
            });
            proj_fwd(c, lin(c, mu, tb + 8), kk, c->vmaps[3 + 4 * l], Sc, (int)R, false, a.U, st);
            c->launch("elem", [&] { launch_vit_gelu(a.U, Sc * R * M, b.A, st); });
            float* Xn = l + 1 < L ? c->vl[l + 1].X : c->vXout;
            proj_fwd(c, lin(c, mu, tb + 10), kk, c->vmaps[4 + 4 * l], Sc, (int)R, false, Xn, st, a.Xmid);
        }
        c->launch("ln", [&] {
            launch_vit_ln_fwd(c->vXout, Sc, B, (int64_t)T * D, RD, D, c->vvec[nt - 4], c->vvec[nt - 3], c->vHcb, D,
                              (int64_t)B * D, c->vstf, st);
        });
        proj_fwd(c, lin(c, mu, nt - 2), kk, c->vmaps[1 + 4 * L], Sc, B, false, c->logits, st);
    }
    // the loss head writes the bf16 seed (GEMM operand) and its fp32 copy (bias gradient)
    c->launch("loss", [&] {
        launch_loss_head(c->logits, Sc, B, c->O, BNN_LOSS_CE, ycls, nullptr, c->vdzb, ldO, true, c->lossrow,
                         c->dz_f32, st);
    });
    c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, st); });
    NvtxRange nvb("bnn.backward");
    auto bias = [&](const SampledLayer& Lb, const float* G, int rows, int64_t ldp, int64_t sG) {
        c->launch("bias", [&] {
            return launch_bias_grad_rows(Lb, kk, Sc, G, rows, (int)ldp, sG, scale, c->vwpart, c->vwpart_cap, c->db_scratch,
                                  acc_mu, acc_rho, st);
        });
    };
    // LayerNorm backward of the token rows: the fused kernel (γ / β chunk sums in place, bf16 copy
    // of dX) when D allows and the chunk sums fit the scratch, else LayerNorm + two row reductions
    const int nq = (int)((R + 63) / 64);
    // (xb: the projection whose output gradient the updated dX is — its bias sums come along)
    const bool fused_ln = vit_ln_bwd_fused_ok(D) && 3 * (int64_t)Sc * nq * D <= c->vwpart_cap;
    auto ln_bwd = [&](const float* dY, const float* Xin, int tv, const float* stats, __nv_bfloat16* dXb,
                      const SampledLayer* xb) {
        if (fused_ln) {
            const int64_t n1 = (int64_t)Sc * nq * D;
            float *pg = c->vwpart, *pb = c->vwpart + n1, *px = xb ? c->vwpart + 2 * n1 : nullptr;
            c->launch("ln", [&] {
                launch_vit_ln_bwd_fused(dY, Xin, Sc, (int)R, D, c->vvec[tv], stats, c->vdX, dXb, pg, pb, px, st);
            });
            c->launch("bias", [&] {
                int nk = 0;
                nk += launch_bias_grad(vec(c, mu, tv), kk, Sc, pg, nq, D, (int64_t)nq * D, scale, c->db_scratch, acc_mu,
                                 acc_rho, st);
                nk += launch_bias_grad(vec(c, mu, tv + 1), kk, Sc, pb, nq, D, (int64_t)nq * D, scale, c->db_scratch, acc_mu,
                                 acc_rho, st);
                if (xb)
                    nk += launch_bias_grad(*xb, kk, Sc, px, nq, D, (int64_t)nq * D, scale, c->db_scratch, acc_mu, acc_rho, st);
                return nk;
            });
            return;
        }
        c->launch("ln", [&] {
            launch_vit_ln_bwd(dY, D, RD, Xin, Sc, (int)R, D, RD, D, c->vvec[tv], stats, c->vdX, c->vdyxh, st);
        });
        bias(vec(c, mu, tv), c->vdyxh, (int)R, D, RD);
        bias(vec(c, mu, tv + 1), dY, (int)R, D, RD);
        if (xb) bias(*xb, c->vdX, (int)R, D, RD);
        if (dXb) c->launch("elem", [&] { launch_vit_cast_bf16(c->vdX, Sc * RD, dXb, st); });
    };
    const bool fused_gelu = M % 4 == 0 && (int64_t)Sc * nq * M <= c->vwpart_cap;
    {
        const SampledLayer Lh = lin(c, mu, nt - 2);
        const WgItem w{Lh, &c->vmaps[1 + 4 * L], 0};
        proj_wgrad(c, kk, Sc, B, scale, acc_mu, acc_rho, &w, 1, st);
        bias(Lh, c->dz_f32, B, c->O, (int64_t)B * c->O);
        proj_dgrad(c, Lh, kk, c->vmaps[1 + 4 * L], Sc, B, c->vdHc, st);
        CUDA_TRY(c, cudaMemsetAsync(c->vdX, 0, sizeof(float) * Sc * RD, st));
        c->launch("ln", [&] {
            launch_vit_ln_bwd(c->vdHc, D, (int64_t)B * D, c->vXout, Sc, B, (int64_t)T * D, RD, D, c->vvec[nt - 4],
                              c->vstf, c->vdX, c->vdyxh, st);
        });
        bias(vec(c, mu, nt - 4), c->vdyxh, B, D, (int64_t)B * D);
        bias(vec(c, mu, nt - 3), c->vdHc, B, D, (int64_t)B * D);
    }
    for (int l = L - 1; l >= 0; --l) {
        bnn_ctx::VitAct& a = c->vl[l];
        const int tb = 4 + 12 * l;
        const SampledLayer Lq = lin(c, mu, tb + 2), Lo = lin(c, mu, tb + 4), L1 = lin(c, mu, tb + 8),
                           L2 = lin(c, mu, tb + 10);
        const bnn_ctx::VitMaps &mq = c->vmaps[1 + 4 * l], &mo = c->vmaps[2 + 4 * l], &m1 = c->vmaps[3 + 4 * l],
                               &m2 = c->vmaps[4 + 4 * l];
        // fc2: G = dX_out (its bf16 copy: from the next layer's LayerNorm-1 backward, or cast here
        // below the final LayerNorm, which touches the cls rows only)
        __nv_bfloat16* dXb_l = (l & 1) ? c->vdXb1 : c->vdXb;
        if (l == L - 1 || !fused_ln) c->launch("elem", [&] { launch_vit_cast_bf16(c->vdX, Sc * RD, dXb_l, st); });
        if (l == L - 1) bias(L2, c->vdX, (int)R, D, RD);  // else: summed by layer l+1's LayerNorm-1 backward
        proj_dgrad(c, L2, kk, m2, Sc, (int)R, c->vdU, st);
        // dU = dA ⊙ GELU'(U): the bf16 GEMM operand, and its fp32 row sums (fc1's bias gradient)
        if (fused_gelu) {
            c->launch("elem", [&] { launch_vit_gelu_bwd_fused(a.U, c->vdU, Sc, (int)R, M, c->vdUb, c->vwpart, st); });
            c->launch("bias", [&] {
                return launch_bias_grad(L1, kk, Sc, c->vwpart, nq, M, (int64_t)nq * M, scale, c->db_scratch, acc_mu, acc_rho,
                                 st);
            });
        } else {
            c->launch("elem", [&] { launch_vit_gelu_bwd_cast(a.U, Sc * R * M, c->vdU, c->vdUb, st); });
            bias(L1, c->vdU, (int)R, M, R * M);
        }
        proj_dgrad(c, L1, kk, m1, Sc, (int)R, c->vdH, st);
        ln_bwd(c->vdH, a.Xmid, tb + 6, a.st2, c->vdXb2, &Lo);  // proj: G = dX_mid (bf16 copy, bias sums)
        proj_dgrad(c, Lo, kk, mo, Sc, (int)R, c->vdO, st);
        c->launch("attn", [&] { launch_vit_attn_bwd_tf32(a.QKV, a.Att, c->vdO, Sc, B, T, D, Hh, c->vdQKV, st); });
        c->launch("elem", [&] { launch_vit_cast_bf16(c->vdQKV, Sc * R * 3 * D, c->vdQKVb, st); });
        bias(Lq, c->vdQKV, (int)R, 3 * D, 3 * RD);
        proj_dgrad(c, Lq, kk, mq, Sc, (int)R, c->vdH, st);
        const SampledLayer L2prev = l > 0 ? lin(c, mu, tb - 12 + 10) : SampledLayer{};  // layer l−1's fc2
        ln_bwd(c->vdH, a.X, tb, a.st1, l > 0 ? ((l & 1) ? c->vdXb : c->vdXb1) : nullptr, l > 0 ? &L2prev : nullptr);
        // the four weight gradients of the layer (their G / X operands are still intact here)
        const WgItem w[4] = {{L2, &m2, 0}, {L1, &m1, 0}, {Lo, &mo, 0}, {Lq, &mq, 0}};
        proj_wgrad(c, kk, Sc, (int)R, scale, acc_mu, acc_rho, w, 4, st);
    }
    bias(vec(c, mu, 2), c->vdX, B, (int64_t)T * D, RD);
    bias(vec(c, mu, 3), c->vdX, B, (int64_t)T * D, RD);
    c->launch("elem", [&] { launch_vit_gather_tokens(c->vdX, Sc, B, T, 1, NP, D, c->vdE, st); });
    c->launch("elem", [&] { launch_vit_cast_bf16(c->vdE, (int64_t)Sc * B * NP * D, c->vdEb, st); });
    const SampledLayer Lp = lin(c, mu, 0);
    const WgItem wp{Lp, &c->vmaps[0], aug ? 0 : 1};
    proj_wgrad(c, kk, Sc, B * NP, scale, acc_mu, acc_rho, &wp, 1, st);
    bias(Lp, c->vdE, B * NP, D, (int64_t)B * NP * D);
    return BNN_OK;
}

int vit_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls, int B, int B_glob, int S_glob,
              int Sc, uint32_t s0, uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss) {
    if (c->bf16)
        return vit_chunk_bf16(c, mu, x, ycls, B, B_glob, S_glob, Sc, s0, seed, step, acc_mu, acc_rho, acc_loss);
    NvtxRange nvtx_("bnn.chunk");
    cudaStream_t st = c->st;
    const SampleKeys kk{make_key(seed), step, s0};
    const int T = c->vT, D = c->vD, M = c->vM, L = c->model.depth, Hh = c->model.heads, NP = c->vNP;
    const int64_t R = (int64_t)B * T, RD = R * D;
    const int nt = (int)c->vtens.size();
    const float scale = 1.0f / ((float)S_glob * B_glob);
    const bool aug = c->cfg.aug == BNN_AUG_PER_SAMPLE;
    const DropArgs nod{};
    const int64_t sP = aug ? (int64_t)B * NP * c->vPK : 0;
    // ---------------- forward
    {
        NvtxRange nv("bnn.forward");
        for (int t = 0; t < nt; ++t)
            if (c->vvec[t])
                c->launch("sample", [&] {
                    launch_vit_sample_vec(mu, c->sigma, c->vtens[t].off, (uint32_t)t, c->vtens[t].cols, kk, Sc,
                                          c->vvec[t], st);
                });
        c->launch("elem", [&] {
            launch_vit_patchify(x, aug ? Sc : 1, B, c->model.in_h, c->model.in_w, c->model.in_c, c->model.patch,
                                aug ? 1 : 0, seed, step, s0, c->gidx * B, c->vP, st);
        });
        const SampledLayer Lp = lin(c, mu, 0);
        c->launch("fwd", [&] {
            launch_fwd_fp32(Lp, kk, nod, Sc, B * NP, c->vP, sP, c->vE, (int64_t)B * NP * D, false, st);
        });
        c->launch("elem", [&] { launch_vit_embed(c->vE, c->vvec[2], c->vvec[3], Sc, B, T, D, c->vX0, st); });
        const float* X = c->vX0;
        for (int l = 0; l < L; ++l) {
            bnn_ctx::VitAct& a = c->vl[l];
            const int tb = 4 + 12 * l;
            c->launch("elem", [&] { cudaMemcpyAsync(a.X, X, sizeof(float) * Sc * RD, cudaMemcpyDeviceToDevice, st); });
            c->launch("ln", [&] {
                launch_vit_ln_fwd(a.X, Sc, (int)R, D, RD, D, c->vvec[tb], c->vvec[tb + 1], a.H1, D, RD, a.st1, st);
            });
            const SampledLayer Lq = lin(c, mu, tb + 2), Lo = lin(c, mu, tb + 4), L1 = lin(c, mu, tb + 8),
                               L2 = lin(c, mu, tb + 10);
            c->launch("fwd", [&] { launch_fwd_fp32(Lq, kk, nod, Sc, (int)R, a.H1, RD, a.QKV, 3 * RD, false, st); });
            c->launch("attn", [&] { launch_vit_attn_fwd(a.QKV, Sc, B, T, D, Hh, a.O, a.Att, st); });
            c->launch("fwd", [&] { launch_fwd_fp32(Lo, kk, nod, Sc, (int)R, a.O, RD, a.Xmid, RD, false, st); });
            c->launch("elem", [&] { launch_vit_add(a.Xmid, a.X, Sc * RD, st); });
            c->launch("ln", [&] {
                launch_vit_ln_fwd(a.Xmid, Sc, (int)R, D, RD, D, c->vvec[tb + 6], c->vvec[tb + 7], a.H2, D, RD, a.st2, st);
            });
            c->launch("fwd", [&] { launch_fwd_fp32(L1, kk, nod, Sc, (int)R, a.H2, RD, a.U, R * M, false, st); });
            c->launch("elem", [&] { launch_vit_gelu(a.U, Sc * R * M, a.A, st); });
            c->launch("fwd", [&] { launch_fwd_fp32(L2, kk, nod, Sc, (int)R, a.A, R * M, c->vXout, RD, false, st); });
            c->launch("elem", [&] { launch_vit_add(c->vXout, a.Xmid, Sc * RD, st); });
            X = c->vXout;
        }
        // final LayerNorm of the cls rows, head, per-sample CE
        c->launch("ln", [&] {
            launch_vit_ln_fwd(c->vXout, Sc, B, (int64_t)T * D, RD, D, c->vvec[nt - 4], c->vvec[nt - 3], c->vHc, D,
                              (int64_t)B * D, c->vstf, st);
        });
        const SampledLayer Lh = lin(c, mu, nt - 2);
        c->launch("fwd", [&] {
            launch_fwd_fp32(Lh, kk, nod, Sc, B, c->vHc, (int64_t)B * D, c->logits, (int64_t)B * c->O, false, st);
        });
    }
    c->launch("loss", [&] {
        launch_loss_head(c->logits, Sc, B, c->O, BNN_LOSS_CE, ycls, nullptr, c->dz_f32, c->O, false, c->lossrow,
                         nullptr, st);
    });
    c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, st); });
    // ---------------- backward
    NvtxRange nvb("bnn.backward");
    auto bias = [&](const SampledLayer& Lb, const float* G, int rows, int64_t ldp, int64_t sG) {
        c->launch("bias", [&] {
            return launch_bias_grad_rows(Lb, kk, Sc, G, rows, (int)ldp, sG, scale, c->vwpart, c->vwpart_cap, c->db_scratch,
                                  acc_mu, acc_rho, st);
        });
    };
    const int nq = (int)((R + 63) / 64);  // LayerNorm backward as in vit_chunk_bf16 (no bf16 copy)
    const bool fused_ln = vit_ln_bwd_fused_ok(D) && 3 * (int64_t)Sc * nq * D <= c->vwpart_cap;
    auto ln_bwd = [&](const float* dY, const float* Xin, int tv, const float* stats) {
        if (fused_ln) {
            float *pg = c->vwpart, *pb = c->vwpart + (int64_t)Sc * nq * D;
            c->launch("ln", [&] {
                launch_vit_ln_bwd_fused(dY, Xin, Sc, (int)R, D, c->vvec[tv], stats, c->vdX, nullptr, pg, pb, nullptr,
                                        st);
            });
            c->launch("bias", [&] {
                int nk = 0;
                nk += launch_bias_grad(vec(c, mu, tv), kk, Sc, pg, nq, D, (int64_t)nq * D, scale, c->db_scratch, acc_mu,
                                 acc_rho, st);
                nk += launch_bias_grad(vec(c, mu, tv + 1), kk, Sc, pb, nq, D, (int64_t)nq * D, scale, c->db_scratch, acc_mu,
                                 acc_rho, st);
                return nk;
            });
            return;
        }
        c->launch("ln", [&] {
            launch_vit_ln_bwd(dY, D, RD, Xin, Sc, (int)R, D, RD, D, c->vvec[tv], stats, c->vdX, c->vdyxh, st);
        });
        bias(vec(c, mu, tv), c->vdyxh, (int)R, D, RD);
        bias(vec(c, mu, tv + 1), dY, (int)R, D, RD);
    };
    {
        const SampledLayer Lh = lin(c, mu, nt - 2);
        c->launch("wgrad", [&] {
            launch_wgrad_fp32(Lh, kk, Sc, B, c->dz_f32, (int64_t)B * c->O, c->vHc, (int64_t)B * D, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap);
        });
        bias(Lh, c->dz_f32, B, c->O, (int64_t)B * c->O);
        c->launch("dgrad", [&] {
            launch_dgrad_fp32(Lh, kk, nod, Sc, B, c->dz_f32, (int64_t)B * c->O, nullptr, 0, c->vdHc, (int64_t)B * D, st);
        });
        CUDA_TRY(c, cudaMemsetAsync(c->vdX, 0, sizeof(float) * Sc * RD, st));
        c->launch("ln", [&] {
            launch_vit_ln_bwd(c->vdHc, D, (int64_t)B * D, c->vXout, Sc, B, (int64_t)T * D, RD, D, c->vvec[nt - 4],
                              c->vstf, c->vdX, c->vdyxh, st);
        });
        bias(vec(c, mu, nt - 4), c->vdyxh, B, D, (int64_t)B * D);
        bias(vec(c, mu, nt - 3), c->vdHc, B, D, (int64_t)B * D);
    }
    for (int l = L - 1; l >= 0; --l) {
        bnn_ctx::VitAct& a = c->vl[l];
        const int tb = 4 + 12 * l;
        const SampledLayer Lq = lin(c, mu, tb + 2), Lo = lin(c, mu, tb + 4), L1 = lin(c, mu, tb + 8),
                           L2 = lin(c, mu, tb + 10);
        // X_out = X_mid + fc2(GELU(fc1(LN2(X_mid))))
        c->launch("wgrad", [&] { launch_wgrad_fp32(L2, kk, Sc, (int)R, c->vdX, RD, a.A, R * M, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap); });
        bias(L2, c->vdX, (int)R, D, RD);
        c->launch("dgrad", [&] { launch_dgrad_fp32(L2, kk, nod, Sc, (int)R, c->vdX, RD, nullptr, 0, c->vdU, R * M, st); });
        c->launch("elem", [&] { launch_vit_gelu_bwd(a.U, Sc * R * M, c->vdU, st); });
        c->launch("wgrad", [&] { launch_wgrad_fp32(L1, kk, Sc, (int)R, c->vdU, R * M, a.H2, RD, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap); });
        bias(L1, c->vdU, (int)R, M, R * M);
        c->launch("dgrad", [&] { launch_dgrad_fp32(L1, kk, nod, Sc, (int)R, c->vdU, R * M, nullptr, 0, c->vdH, RD, st); });
        ln_bwd(c->vdH, a.Xmid, tb + 6, a.st2);
        // X_mid = X + proj(attention(LN1(X)))
        c->launch("wgrad", [&] { launch_wgrad_fp32(Lo, kk, Sc, (int)R, c->vdX, RD, a.O, RD, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap); });
        bias(Lo, c->vdX, (int)R, D, RD);
        c->launch("dgrad", [&] { launch_dgrad_fp32(Lo, kk, nod, Sc, (int)R, c->vdX, RD, nullptr, 0, c->vdO, RD, st); });
        c->launch("attn", [&] { launch_vit_attn_bwd(a.QKV, a.Att, c->vdO, Sc, B, T, D, Hh, c->vdQKV, st); });
        c->launch("wgrad", [&] { launch_wgrad_fp32(Lq, kk, Sc, (int)R, c->vdQKV, 3 * RD, a.H1, RD, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap); });
        bias(Lq, c->vdQKV, (int)R, 3 * D, 3 * RD);
        c->launch("dgrad", [&] { launch_dgrad_fp32(Lq, kk, nod, Sc, (int)R, c->vdQKV, 3 * RD, nullptr, 0, c->vdH, RD, st); });
        ln_bwd(c->vdH, a.X, tb, a.st1);
    }
    // X_0 = [cls; patch·W_pᵀ + b_p] + pos
    bias(vec(c, mu, 2), c->vdX, B, (int64_t)T * D, RD);  // cls: token-0 rows
    {
        SampledLayer Lpos = vec(c, mu, 3);  // pos [1, T·D]: Σ over the B examples of the whole [T·D] row
        bias(Lpos, c->vdX, B, (int64_t)T * D, RD);
    }
    c->launch("elem", [&] { launch_vit_gather_tokens(c->vdX, Sc, B, T, 1, NP, D, c->vdE, st); });
    const SampledLayer Lp = lin(c, mu, 0);
    c->launch("wgrad", [&] {
        launch_wgrad_fp32(Lp, kk, Sc, B * NP, c->vdE, (int64_t)B * NP * D, c->vP, sP, scale, acc_mu, acc_rho, st, c->vwpart, c->vwpart_cap);
    });
    bias(Lp, c->vdE, B * NP, D, (int64_t)B * NP * D);
    return BNN_OK;
}
