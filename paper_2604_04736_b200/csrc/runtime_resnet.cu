// runtime_resnet.cu — BF16 orchestration of the ResNet-18-shaped Bayesian CNN (C3–C5).
//
// Per sample chunk (SURVEY.md §3.3 with the conv kernels of kernels_conv_tc.cu):
//   input (K9 augmentation, bf16, channels padded to 8)
//   → for each conv: W_s scratch (one layer, all chunk samples) → tcgen05 implicit-GEMM fwd
//     with bias / residual / ReLU fused
//   → GAP → linear head (the MLP generator kernel) → loss head
//   → head wgrad/dgrad → GAP backward (+ReLU mask, bias partials)
//   → for each conv in reverse: bias grad from fused partials, tcgen05 wgrad with the
//     ε-regenerating sample-accumulating epilogue, W_s regenerated → tcgen05 dgrad with the
//     residual contribution, the ReLU mask of the layer input and the producer's bias partials
//     fused into the epilogue.
#include "ctx.cuh"
#include "common.cuh"

namespace {

bool is_fc(const bnn_ctx* c, const ROp& op) { return op.type == 0 && op.dst == c->rlogits; }

// a 1×1 projection's output sc is the only conv output without ReLU (besides the head)
bool is_proj_output(const bnn_ctx* c, int buf) {
    for (const ROp& p : c->rops)
        if (p.type == 0 && p.dst == buf && p.relu == 0 && !is_fc(c, p)) return true;
    return false;
}

// buffer whose gradient is "dL/d(this op's pre-activation output)": the op's own output,
// except for a projection, whose output sc is summed into the block output y
// stage-1 64 → 64 stride-1 3×3 convs on the W-stationary row-packed kernels (kernels_conv64.cu);
// BNN_CONV_HALO=0 or BNN_CONV64=0 puts them back on conv3's tiles, BNN_CONV64W=0 their weight
// gradients back on the generic conv2 wgrad
static bool env_on(const char* name) {
    const char* e = getenv(name);
    return !(e && atoi(e) == 0);
}
bool conv64_layer(const bnn_ctx* c, const ROp& op) {
    if (op.type != 0 || is_fc(c, op) || op.src == 0 || !env_on("BNN_CONV_HALO") || !env_on("BNN_CONV64")) return false;
    const LayerDesc& Ld = c->layers[op.layer];
    const RBuf& Sb = c->rbufs[op.src];
    const RBuf& Db = c->rbufs[op.dst];
    return Ld.stride == 1 && Ld.k == 3 && Ld.pad == 1 && Ld.cin == 64 && Ld.cout == 64 && Sb.C == 64 &&
           Db.C == 64 && c->rbf[op.src].C_pad == 64 && Db.H == Sb.H && Db.W == Sb.W && conv64_ok(Db.H, Db.W);
}
bool conv64w_layer(const bnn_ctx* c, const ROp& op) {
    return conv64_layer(c, op) && env_on("BNN_CONV64W") && conv64_wgrad_ok(c->rbufs[op.dst].H, c->rbufs[op.dst].W);
}
// ε-fused sample accumulation in the weight-gradient kernel (clusters of the chunk's samples):
// the number of pixel splits (co-resident clusters), or 0 for the per-sample partials + ε combine
int eps_fused_nsplit(const bnn_ctx* c, const ROp& op, int Sc) {
    if (!conv64w_layer(c, op) || !env_on("BNN_WGRAD_EPS")) return 0;
    const int Gc = conv64_wgrad_eps_cluster(Sc);
    return conv64_wgrad_eps_nsplit(Sc, Gc) / (Sc / Gc);  // pixel splits (partials = splits × sample groups)
}

int grad_src_buffer(const bnn_ctx* c, int dst) {
    if (is_proj_output(c, dst))
        for (const ROp& op : c->rops)
            if (op.type == 0 && op.res == dst) return op.dst;
    return dst;
}

}  // namespace

int alloc_resnet_bf16(bnn_ctx* c) {
    const int B = c->B_max, Sc = c->chunk;
    const int bw = c->layers[0].cout;
    if (bw % 64 != 0)
        return c->set_err(BNN_ERR_CONFIG, "BF16 ResNet needs base_width %% 64 == 0 (tcgen05 conv tiles)");
    if (c->rbufs[0].H % 8 != 0 || c->rbufs[0].W % 8 != 0)
        return c->set_err(BNN_ERR_CONFIG, "ResNet input H, W must be multiples of 8 (three stride-2 stages)");
    const int nb = (int)c->rbufs.size();
    c->rbf.assign(nb, bnn_ctx::RBf{});
    for (int i = 0; i < nb; ++i) c->rbf[i].C_pad = i == 0 ? (int)round_up(c->rbufs[0].C, 8) : c->rbufs[i].C;
    const int gbuf = c->rops[c->rops.size() - 2].dst;  // GAP output (pooled features)
    for (int i = 0; i < nb; ++i) {
        if (i == c->rlogits) continue;
        const RBuf& R = c->rbufs[i];
        bnn_ctx::RBf& b = c->rbf[i];
        const size_t n = (size_t)Sc * B * R.H * R.W * b.C_pad;
        if (!c->alloc(&b.val, n)) return c->set_err(BNN_ERR_CUDA, "out of memory (activations)");
        if (i != 0 && !c->alloc(&b.grad, n)) return c->set_err(BNN_ERR_CUDA, "out of memory (gradients)");
        if (i != 0 && i != gbuf && R.C % 32 == 0 && c->rbufs[i].H > 1) {
            if (!c->alloc(&b.mbits, n / 32)) return c->set_err(BNN_ERR_CUDA, "out of memory (masks)");
        }
        if (i != 0 && i != gbuf) {
            const int64_t npix = (int64_t)B * R.H * R.W;
            b.bpart_cap = (int64_t)(4 * ((npix + 127) / 128) * 4 + B) * R.C;
            if (!c->alloc(&b.bpart, (size_t)Sc * b.bpart_cap)) return c->set_err(BNN_ERR_CUDA, "out of memory");
        }
    }
    const int O = c->O;
    if (!c->alloc(&c->logits, (size_t)Sc * B * O) || !c->alloc(&c->lossrow, (size_t)Sc * B) ||
        !c->alloc(&c->dz_f32, (size_t)Sc * B * O) || !c->alloc(&c->fcG, (size_t)Sc * B * round_up(O, 8)))
        return c->set_err(BNN_ERR_CUDA, "out of memory (head)");
    // per-layer geometry, scratch sizes and TMA descriptors
    const int L = (int)c->layers.size();
    c->kpad.assign(L, 0);
    c->wscr_off.assign(L, 0);
    c->nsplit.assign(L, 1);
    c->wgrad_eps.assign(L, 0);
    c->wcps.assign(L, 1);
    c->wkpx.assign(L, 64);
    c->cmap_w.resize(L);
    c->cmap_wT.resize(L);
    c->cmap_g.resize(L);
    c->cmap_bf.resize(L);
    c->cmap_bd.resize(L);
    c->cmap_xw.resize(L);
    c->cmap_a2f.resize(L);
    c->cmap_a2d.resize(L);
    c->cmap_w2.resize(L);
    c->cmap_w64.resize(L);
    c->tma_a2f.assign(L, 0);
    c->tma_a2d.assign(L, 0);
    c->tma_fwd.assign(L, 0);
    c->tma_dgrad.assign(L, 0);
    c->tma_wgrad.assign(L, 0);
    size_t wmax = 0, pmax = 0;
    int maxN = 0;
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const int Cp = c->rbf[op.src].C_pad, taps = Ld.k * Ld.k;
        const int Kp = (int)round_up((int64_t)taps * Cp, 64);
        c->kpad[op.layer] = Kp;
        c->wscr_off[op.layer] = wmax;
        wmax += round_up((int64_t)Sc * Ld.cout * Kp, 512);
        maxN = std::max(maxN, Ld.cout);
        const RBuf& D = c->rbufs[op.dst];
        const int64_t npix = (int64_t)B * D.H * D.W;
        const int Cp_src = c->rbf[op.src].C_pad;
        if (Ld.cin % 64 == 0 || Cp_src == 8) {  // conv2 wgrad: units = samples × splits × co tiles × column tiles
            const int Kt = conv2_wgrad_cols(taps, Ld.cin, Cp_src);
            const int base = Sc * ((Ld.cout + 127) / 128) * ((Kt + 255) / 256);
            // 64-channel layers on the TMA operand path: 128-pixel k-steps halve the TMA ops
            {
                const RBuf& Sb0 = c->rbufs[op.src];
                const int PW = D.W, PH = D.H, kp = 128;
                const int wh = PW >= kp ? 1 : std::min(PH, kp / PW);
                const bool shared = op.src == 0 && c->cfg.aug != BNN_AUG_PER_SAMPLE;
                // stride 2: the same with the element-stride-2 X window (stage-3 stride-2 wgrad 85 → 76 µs;
                // BNN_WGRAD_S2_KP128=0 keeps 64-pixel k-steps there)
                const bool s2 = Ld.stride == 2 && Sb0.W == 2 * PW && op.src != 0 && Cp_src == Ld.cin &&
                                env_on("BNN_WGRAD_S2_TMA") && env_on("BNN_WGRAD_S2_KP128");
                if ((Ld.stride == 1 && Sb0.W == PW || s2) && Ld.cout <= 512 && Ld.cin % 64 == 0 && !shared &&
                    kp % PW == 0 && PH % wh == 0 && (kp / (PW * wh)) * PW * wh == kp)
                    c->wkpx[op.layer] = kp;
            }
            // CTAs per SM of the conv2 weight gradient (measured per stage, C3): two (64-pixel k-steps)
            // for the gather-path layers (stride 2, the stem) and the ≤ 2048-pixel-per-sample layers
            // (stage 4: 91 → 85 µs, the stride-2 ones 102 → 82, 135 → 124); one with 128-pixel k-steps
            // for stages 2 and 3 (two CTAs there: 77 → 108, 92 → 100)
            {
                const int forced = conv2_wgrad_cps();
                const bool two = forced ? forced == 2 : (c->wkpx[op.layer] == 64 || npix <= 2048);
                c->wcps[op.layer] = two ? 2 : 1;
                if (two) c->wkpx[op.layer] = 64;
            }
            const int blocks = (int)((npix + c->wkpx[op.layer] - 1) / c->wkpx[op.layer]);
            const int epsn = eps_fused_nsplit(c, op, Sc);
            c->wgrad_eps[op.layer] = epsn > 0 ? 1 : 0;
            c->nsplit[op.layer] = epsn > 0 ? epsn : conv64w_layer(c, op) ? conv64_wgrad_nsplit(Sc) : conv2_wgrad_nsplit(base, blocks, c->wcps[op.layer]);
            if (Ld.off_w % 4 != 0) return c->set_err(BNN_ERR_CONFIG, "conv weight offset not 16-byte aligned");
            // per-sample partials [s][split][co][cols], or (ε-fused) partials [split·group][μ | ρ][co·cols]
            // (≤ Sc sample groups for any chunk size)
            pmax = std::max(pmax, (size_t)(epsn > 0 ? 2 * Sc : Sc) * c->nsplit[op.layer] * Ld.cout * Kt);
            continue;
        } else {  // SIMT wgrad (the stem): split pixels so ≥ 2 waves of CTAs exist
            const int tiles = (int)(((int64_t)taps * Ld.cin + 63) / 64) * ((Ld.cout + 63) / 64);
            c->nsplit[op.layer] = (int)std::max<int64_t>(1, std::min<int64_t>((npix + 255) / 256,
                                                                              (8 * bnn::kNumSMs) / tiles));
        }
        pmax = std::max(pmax, (size_t)c->nsplit[op.layer] * 2 * Ld.cout * taps * Ld.cin);
    }
    c->bias_rows_cap = (int64_t)Sc * 64 * std::max(maxN, O);
    if (!c->alloc(&c->wscr, wmax) || !c->alloc(&c->wpart, std::max<size_t>(pmax, 1)) ||
        !c->alloc(&c->wpart2, std::max<size_t>(pmax, 1)) ||
        !c->alloc(&c->bias_scr, (size_t)Sc * 512 * c->layers.size()) ||  // one slot per layer
        !c->alloc(&c->db_scratch, (size_t)2 * Sc * std::max(maxN, O)) ||
        !c->alloc(&c->bias_rows_scr, (size_t)Sc * 64 * std::max(maxN, O)))
        return c->set_err(BNN_ERR_CUDA, "out of memory (scratch)");
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const int Kp = c->kpad[op.layer], CO = Ld.cout, taps = Ld.k * Ld.k;
        {
            const uint64_t dims[3] = {(uint64_t)Kp, (uint64_t)CO, (uint64_t)Sc};
            const uint64_t str[2] = {(uint64_t)Kp * 2, (uint64_t)CO * Kp * 2};
            const uint32_t box[3] = {64, 128, 1};
            if (!make_map_nd(&c->cmap_w[op.layer], c->wscr + c->wscr_off[op.layer], 3, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (W scratch) failed");
            const uint32_t box64[3] = {64, 64, 1};
            if (!make_map_nd(&c->cmap_w64[op.layer], c->wscr + c->wscr_off[op.layer], 3, dims, str, box64))
                return c->set_err(BNN_ERR_CUDA, "tensor map (W scratch, 64 rows) failed");
            const uint32_t box2[3] = {64, (uint32_t)std::min(CO, 256), 1};
            if (!make_map_nd(&c->cmap_w2[op.layer], c->wscr + c->wscr_off[op.layer], 3, dims, str, box2))
                return c->set_err(BNN_ERR_CUDA, "tensor map (W scratch, conv2) failed");
        }
        if (Ld.cin % 64 == 0 || c->rbf[op.src].C_pad == 8) {
            const int gb = grad_src_buffer(c, op.dst);
            const RBuf& D = c->rbufs[op.dst];
            const uint64_t npix = (uint64_t)B * D.H * D.W;
            // dY as (64 co, pixel, co block, sample): one op loads 64 pixels × 128 co
            const uint64_t gd[4] = {64, npix, (uint64_t)(CO / 64), (uint64_t)Sc};
            const uint64_t gs[3] = {(uint64_t)CO * 2, 128, npix * CO * 2};
            const uint32_t gbx[4] = {64, (uint32_t)c->wkpx[op.layer], (uint32_t)std::min(2, CO / 64), 1};
            if (!make_map_nd(&c->cmap_g[op.layer], c->rbf[gb].grad, 4, gd, gs, gbx))
                return c->set_err(BNN_ERR_CUDA, "tensor map (dY) failed");
        }
        if (Ld.cin % 64 == 0) {
            // W_sᵀ as (64 ci, tap, co, ci block, sample): one op loads cb blocks of 64 ci × 64 co
            const int cb = Ld.cin <= 128 ? std::min(2, Ld.cin / 64) : std::min(Ld.cin, 256) / 64;  // 1: conv3 dup
            const uint64_t dims[5] = {64, (uint64_t)taps, (uint64_t)CO, (uint64_t)(Ld.cin / 64), (uint64_t)Sc};
            const uint64_t str[4] = {(uint64_t)Ld.cin * 2, (uint64_t)Kp * 2, 128, (uint64_t)CO * Kp * 2};
            const uint32_t box[5] = {64, 1, 64, (uint32_t)cb, 1};
            if (!make_map_nd(&c->cmap_wT[op.layer], c->wscr + c->wscr_off[op.layer], 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (W scratch transposed) failed");
        }
    }
    // stride-1 convs: the B operand (activation / dY window) by 5-D TMA with OOB zero fill
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        if (Ld.stride != 1) continue;
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        const int PW = Db.W, PH = Db.H;  // stride 1: output pixel space == input pixel space
        if (256 % PW != 0) continue;
        const int th = std::min(PH, 256 / PW);
        if (PH % th != 0) continue;
        const int tn = 256 / (PW * th);
        const uint32_t box[5] = {64, (uint32_t)PW, (uint32_t)th, (uint32_t)tn, 1};
        const int Cp = c->rbf[op.src].C_pad;
        if (Cp % 64 == 0) {
            const bool shared = op.src == 0 && c->cfg.aug != BNN_AUG_PER_SAMPLE;
            const uint64_t dims[5] = {(uint64_t)Cp, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B,
                                      (uint64_t)(shared ? 1 : Sc)};
            const uint64_t str[4] = {(uint64_t)Cp * 2, (uint64_t)Sb.W * Cp * 2, (uint64_t)Sb.H * Sb.W * Cp * 2,
                                     (uint64_t)B * Sb.H * Sb.W * Cp * 2};
            if (!make_map_nd(&c->cmap_bf[op.layer], c->rbf[op.src].val, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (activation window) failed");
            c->tma_fwd[op.layer] = 1;
            // wgrad: 64-pixel blocks of the output pixel space
            if (64 % PW == 0 || PW % 64 == 0) {
                const int kp = c->wkpx[op.layer];
                const int wh = PW >= kp ? 1 : std::min(PH, kp / PW);
                const int wn = kp / (std::min(PW, kp) * wh);
                if (PW <= 64 && PH % wh == 0 && wn >= 1 && !shared) {
                    // X as (64 ci, W, H, image·sample, ci block): one op loads cbx channel blocks
                    const int Kt = Ld.k * Ld.k * Ld.cin;
                    const int cbx = std::min(4, Ld.cin / 64);  // divides every column tile's block count
                    (void)Kt;
                    const uint64_t xd[5] = {64, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B * Sc, (uint64_t)(Cp / 64)};
                    const uint64_t xs[4] = {(uint64_t)Cp * 2, (uint64_t)Sb.W * Cp * 2, (uint64_t)Sb.H * Sb.W * Cp * 2, 128};
                    const uint32_t wbox[5] = {64, (uint32_t)std::min(PW, kp), (uint32_t)wh, (uint32_t)wn, (uint32_t)cbx};
                    if (!make_map_nd(&c->cmap_xw[op.layer], c->rbf[op.src].val, 5, xd, xs, wbox))
                        return c->set_err(BNN_ERR_CUDA, "tensor map (wgrad window) failed");
                    c->tma_wgrad[op.layer] = Ld.cin % 64 == 0 ? 1 : 0;
                }
            }
        }
        if (op.src != 0 && Db.C % 64 == 0 && Ld.cin % 64 == 0) {
            const int gb = grad_src_buffer(c, op.dst);
            const uint64_t dims[5] = {(uint64_t)Db.C, (uint64_t)Db.W, (uint64_t)Db.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {(uint64_t)Db.C * 2, (uint64_t)Db.W * Db.C * 2,
                                     (uint64_t)Db.H * Db.W * Db.C * 2, (uint64_t)B * Db.H * Db.W * Db.C * 2};
            if (!make_map_nd(&c->cmap_bd[op.layer], c->rbf[gb].grad, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (dY window) failed");
            c->tma_dgrad[op.layer] = 1;
        }
    }
    // conv3 HALO (stride-1 3×3 layers with 64-channel B operands, kernels_conv2.cu): one padded
    // row (W + 2 pixels, OOB columns / rows zero-filled) per TMA box; BNN_CONV_HALO=0 disables
    c->cmap_hf.resize(L);
    c->cmap_hd.resize(L);
    c->halo_fwd.assign(L, 0);
    c->halo_dgrad.assign(L, 0);
    c->conv64.assign(L, 0);
    c->rowmaps.resize(L);
    const char* he = getenv("BNN_CONV_HALO");
    const bool halo_on = !(he && atoi(he) == 0);
    for (const ROp& op : c->rops) {
        if (!halo_on || op.type != 0 || is_fc(c, op) || op.src == 0) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        if (Ld.stride != 1 || Ld.k != 3 || Ld.pad != 1 || !conv3_halo_ok(Db.H, Db.W)) continue;
        const uint32_t box[5] = {64, (uint32_t)(Db.W + 2), 1, 1, 1};
        if (c->rbf[op.src].C_pad == 64 && Db.C <= 128) {  // fwd: conv3 with a 64-channel input window
            const uint64_t dims[5] = {64, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {128, (uint64_t)Sb.W * 128, (uint64_t)Sb.H * Sb.W * 128,
                                     (uint64_t)B * Sb.H * Sb.W * 128};
            if (!make_map_nd(&c->cmap_hf[op.layer], c->rbf[op.src].val, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (conv3 halo window) failed");
            c->halo_fwd[op.layer] = 1;
        }
        if (Db.C == 64 && Sb.C <= 128 && Ld.cin % 64 == 0) {  // dgrad: conv3 over a 64-channel dY window
            const int gb = grad_src_buffer(c, op.dst);
            const uint64_t dims[5] = {64, (uint64_t)Db.W, (uint64_t)Db.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {128, (uint64_t)Db.W * 128, (uint64_t)Db.H * Db.W * 128,
                                     (uint64_t)B * Db.H * Db.W * 128};
            if (!make_map_nd(&c->cmap_hd[op.layer], c->rbf[gb].grad, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (conv3 halo dY window) failed");
            c->halo_dgrad[op.layer] = 1;
        }
        // both directions 64 → 64 (stage 1): the W-stationary row-packed kernel (kernels_conv64.cu)
        if (conv64_layer(c, op) && c->halo_fwd[op.layer] && c->halo_dgrad[op.layer]) {
            c->conv64[op.layer] = 1;
            // the weight gradient's dY / X row runs: boxes of 1 … 8 padded rows (W + 2 pixels each)
            const int gb = grad_src_buffer(c, op.dst);
            const uint64_t dims[5] = {64, (uint64_t)Db.W, (uint64_t)Db.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {128, (uint64_t)Db.W * 128, (uint64_t)Db.H * Db.W * 128,
                                     (uint64_t)B * Db.H * Db.W * 128};
            for (int h = 1; h <= 8; ++h) {
                const uint32_t bx[5] = {64, (uint32_t)(Db.W + 2), (uint32_t)std::min(h, Db.H), 1, 1};
                if (!make_map_nd(&c->rowmaps[op.layer].y[h - 1], c->rbf[gb].grad, 5, dims, str, bx) ||
                    !make_map_nd(&c->rowmaps[op.layer].x[h - 1], c->rbf[op.src].val, 5, dims, str, bx))
                    return c->set_err(BNN_ERR_CUDA, "tensor map (conv64 weight-gradient rows) failed");
            }
        }
    }
    // the stem (kernels_stem.cu): the 8-channel input as 1-row boxes of W + 2 pixels (OOB zero
    // columns), no swizzle (16-byte rows: the MMA's two K core matrices are two taps)
    c->stem_layer = -1;
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op) || op.src != 0 || !env_on("BNN_STEM")) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        if (Ld.k != 3 || Ld.stride != 1 || Ld.pad != 1 || c->rbf[0].C_pad != 8 || Ld.cout != 64 || op.res >= 0 ||
            !op.relu || Db.H != Sb.H || Db.W != Sb.W)
            continue;
        const bool shared = c->cfg.aug != BNN_AUG_PER_SAMPLE;
        const uint64_t dims[5] = {8, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B, (uint64_t)(shared ? 1 : Sc)};
        const uint64_t str[4] = {16, (uint64_t)Sb.W * 16, (uint64_t)Sb.H * Sb.W * 16, (uint64_t)B * Sb.H * Sb.W * 16};
        bool ok = true;
        for (int h = 1; h <= 8; ++h) {
            const uint32_t box[5] = {8, (uint32_t)stem_row_pitch(Sb.W), (uint32_t)std::min(h, Sb.H), 1, 1};
            ok = ok && make_map_nd(&c->cmap_stem.x[h - 1], c->rbf[0].val, 5, dims, str, box, nullptr,
                                   CU_TENSOR_MAP_SWIZZLE_NONE);
        }
        if (ok) c->stem_layer = op.layer;
    }
    // stride-2 forward: the input window of a 2-strided conv is a TMA box with element stride 2
    // in W and H (box = 2·extent raw elements, every other one loaded); conv3 256-pixel and
    // conv2 128-pixel tiles of the output grid
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op) || op.src == 0) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        const int Cp = c->rbf[op.src].C_pad;
        if (Ld.stride != 2 || Cp % 64 != 0) continue;
        const int PW = Db.W, PH = Db.H;
        for (int px : {256, 128}) {
            if (px % PW != 0 || 2 * PW > 256) continue;
            const int th = std::min(PH, px / PW);
            if (PH % th != 0 || 2 * th > 256) continue;
            const uint32_t box[5] = {64, (uint32_t)(2 * PW), (uint32_t)(2 * th), (uint32_t)(px / (PW * th)), 1};
            const uint32_t es[5] = {1, 2, 2, 1, 1};
            const uint64_t dims[5] = {(uint64_t)Cp, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {(uint64_t)Cp * 2, (uint64_t)Sb.W * Cp * 2, (uint64_t)Sb.H * Sb.W * Cp * 2,
                                     (uint64_t)B * Sb.H * Sb.W * Cp * 2};
            CUtensorMap* m = px == 256 ? &c->cmap_bf[op.layer] : &c->cmap_a2f[op.layer];
            if (!make_map_nd(m, c->rbf[op.src].val, 5, dims, str, box, es))
                return c->set_err(BNN_ERR_CUDA, "tensor map (stride-2 activation window) failed");
            (px == 256 ? c->tma_fwd : c->tma_a2f)[op.layer] = 1;
        }
        // weight gradient: the X window of a 64-pixel k-step (whole output rows) with the same
        // element stride 2, one op per run of channel blocks of a tap (as the stride-1 map above)
        const int kp = c->wkpx[op.layer];
        const int wh = PW >= kp ? 1 : std::min(PH, kp / PW);
        const int wn = kp / (std::min(PW, kp) * wh);
        if (env_on("BNN_WGRAD_S2_TMA") && (kp == 64 || kp == 128) && PW <= 64 && kp % PW == 0 && PH % wh == 0 && wn >= 1 &&
            Ld.cin % 64 == 0 && Cp == Ld.cin) {
            const int cbx = std::min(4, Ld.cin / 64);
            const uint64_t xd[5] = {64, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B * Sc, (uint64_t)(Cp / 64)};
            const uint64_t xs[4] = {(uint64_t)Cp * 2, (uint64_t)Sb.W * Cp * 2, (uint64_t)Sb.H * Sb.W * Cp * 2, 128};
            const uint32_t wbox[5] = {64, (uint32_t)(2 * std::min(PW, kp)), (uint32_t)(2 * wh), (uint32_t)wn,
                                      (uint32_t)cbx};
            const uint32_t wes[5] = {1, 2, 2, 1, 1};
            if (!make_map_nd(&c->cmap_xw[op.layer], c->rbf[op.src].val, 5, xd, xs, wbox, wes))
                return c->set_err(BNN_ERR_CUDA, "tensor map (stride-2 wgrad window) failed");
            c->tma_wgrad[op.layer] = 1;
        }
    }
    // stride-2 dgrad: each input-pixel parity class reads a plain shifted window of dY over the
    // output grid, so dY windows by TMA too (conv3: 256-pixel box; conv2: 128-pixel box below)
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op) || op.src == 0) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        if (Ld.stride != 2 || Sb.H != 2 * Db.H || Sb.W != 2 * Db.W) continue;
        if (Db.C % 64 != 0 || Ld.cin % 64 != 0 || Sb.C > 128) continue;
        const int PW = Db.W, PH = Db.H;
        if (256 % PW != 0) continue;
        const int th = std::min(PH, 256 / PW);
        if (PH % th != 0) continue;
        const uint32_t box[5] = {64, (uint32_t)PW, (uint32_t)th, (uint32_t)(256 / (PW * th)), 1};
        const int gb = grad_src_buffer(c, op.dst);
        const uint64_t dims[5] = {(uint64_t)Db.C, (uint64_t)Db.W, (uint64_t)Db.H, (uint64_t)B, (uint64_t)Sc};
        const uint64_t str[4] = {(uint64_t)Db.C * 2, (uint64_t)Db.W * Db.C * 2, (uint64_t)Db.H * Db.W * Db.C * 2,
                                 (uint64_t)B * Db.H * Db.W * Db.C * 2};
        if (!make_map_nd(&c->cmap_bd[op.layer], c->rbf[gb].grad, 5, dims, str, box))
            return c->set_err(BNN_ERR_CUDA, "tensor map (stride-2 dY window) failed");
        c->tma_dgrad[op.layer] = 1;
    }
    // conv2: 128-pixel windows for the A operand (activation: stride 1; dY: stride 1 and 2)
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        // stride 1: activation and dY windows; stride 2 (Sb = 2·Db): the dY window of each
        // input-pixel parity class (the forward's strided input stays a gather)
        const bool s1 = Ld.stride == 1;
        if (!s1 && (Ld.stride != 2 || Sb.H != 2 * Db.H || Sb.W != 2 * Db.W)) continue;
        const int PW = Db.W, PH = Db.H;
        if (128 % PW != 0) continue;
        const int th = std::min(PH, 128 / PW);
        if (PH % th != 0) continue;
        const int tn = 128 / (PW * th);
        const uint32_t box[5] = {64, (uint32_t)PW, (uint32_t)th, (uint32_t)tn, 1};
        const int Cp = c->rbf[op.src].C_pad;
        if (s1 && Cp % 64 == 0) {
            const bool shared = op.src == 0 && c->cfg.aug != BNN_AUG_PER_SAMPLE;
            const uint64_t dims[5] = {(uint64_t)Cp, (uint64_t)Sb.W, (uint64_t)Sb.H, (uint64_t)B,
                                      (uint64_t)(shared ? 1 : Sc)};
            const uint64_t str[4] = {(uint64_t)Cp * 2, (uint64_t)Sb.W * Cp * 2, (uint64_t)Sb.H * Sb.W * Cp * 2,
                                     (uint64_t)B * Sb.H * Sb.W * Cp * 2};
            if (!make_map_nd(&c->cmap_a2f[op.layer], c->rbf[op.src].val, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (conv2 activation window) failed");
            c->tma_a2f[op.layer] = 1;
        }
        if (op.src != 0 && Db.C % 64 == 0 && Ld.cin % 64 == 0) {
            const int gb = grad_src_buffer(c, op.dst);
            const uint64_t dims[5] = {(uint64_t)Db.C, (uint64_t)Db.W, (uint64_t)Db.H, (uint64_t)B, (uint64_t)Sc};
            const uint64_t str[4] = {(uint64_t)Db.C * 2, (uint64_t)Db.W * Db.C * 2,
                                     (uint64_t)Db.H * Db.W * Db.C * 2, (uint64_t)B * Db.H * Db.W * Db.C * 2};
            if (!make_map_nd(&c->cmap_a2d[op.layer], c->rbf[gb].grad, 5, dims, str, box))
                return c->set_err(BNN_ERR_CUDA, "tensor map (conv2 dY window) failed");
            c->tma_a2d[op.layer] = 1;
        }
    }
    if (cudaStreamCreateWithFlags(&c->side3, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join3, cudaEventDisableTiming) != cudaSuccess)
        return c->set_err(BNN_ERR_CUDA, "stream creation failed");
    for (int i = 0; i < 2; ++i)
        if (cudaEventCreateWithFlags(&c->ev_wg[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_comb[i], cudaEventDisableTiming) != cudaSuccess)
            return c->set_err(BNN_ERR_CUDA, "event creation failed");
    // one event per layer: its W_s slot is written (the side stream generates ahead)
    c->wgen_ev.assign(c->layers.size(), nullptr);
    for (auto& e : c->wgen_ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            return c->set_err(BNN_ERR_CUDA, "event creation failed");
    // head: pooled features [S][B][Cf] → logits, with the MLP kernels' descriptors
    const int Cf = c->rbufs[gbuf].C, ldO = (int)round_up(O, 8);
    c->map_fwdB.resize(1);
    c->map_dgradB.resize(1);
    c->map_wgG.resize(1);
    c->map_wgX.resize(1);
    if (!make_map(&c->map_fwdB[0], c->rbf[gbuf].val, Cf, B, Sc, Cf, 256) ||
        !make_map(&c->map_wgX[0], c->rbf[gbuf].val, Cf, B, Sc, Cf, 64) ||
        !make_map(&c->map_dgradB[0], c->fcG, O, B, Sc, ldO, 256) ||
        !make_map(&c->map_wgG[0], c->fcG, O, B, Sc, ldO, 64))
        return c->set_err(BNN_ERR_CUDA, "tensor map (head) failed");
    c->map_B = B;
    return BNN_OK;
}

void resnet_bf16_forward(bnn_ctx* c, const float* mu, const float* x, int Sc, int B, uint64_t seed,
                         uint32_t step, uint32_t s0, bool aug) {
    cudaStream_t st = c->st;
    SampleKeys kk{make_key(seed), step, s0};
    const RBuf& in = c->rbufs[0];
    const int Cp0 = c->rbf[0].C_pad;
    c->launch("aug", [&] {
        launch_input_bf16(x, aug ? Sc : 1, B, in.H, in.W, in.C, Cp0, aug ? 1 : 0, seed, step, s0,
                          c->gidx * B, c->rbf[0].val, st);
    });
    const int64_t in_stride = aug ? (int64_t)B * in.H * in.W * Cp0 : 0;
    // every conv layer's W_s slot and sampled biases, generated ahead on the side stream in
    // layer order (they depend on σ only); the forward conv of layer l waits for its event
    const bool ahead = !c->prof && c->side;
    cudaStream_t ss = fork_side(c);
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        SampledLayer sl = sampled(c, op.layer, mu);
        const LayerDesc& Ld = c->layers[op.layer];
        const int Cp = c->rbf[op.src].C_pad;
        c->launch("wgen", [&] {
            launch_gen_wscratch(sl, kk, Sc, Ld.cin, Cp, Ld.k * Ld.k, c->kpad[op.layer], c->wscr + c->wscr_off[op.layer],
                                c->bias_scr + (size_t)op.layer * Sc * 512, ss);
        });
        if (ahead) cudaEventRecord(c->wgen_ev[op.layer], ss);
    }
    for (const ROp& op : c->rops) {
        if (op.type == 1) {
            const RBuf& S = c->rbufs[op.src];
            c->launch("gap", [&] {
                launch_gap_fwd_bf16(c->rbf[op.src].val, Sc * B, S.H * S.W, S.C, c->rbf[op.dst].val, st);
            });
            continue;
        }
        SampledLayer sl = sampled(c, op.layer, mu);
        if (is_fc(c, op)) {
            TcGenArgs a{};
            a.L = sl;
            a.kk = kk;
            a.mode = 0;
            a.B = B;
            a.b_shared = 0;
            a.M = sl.N;
            a.R = sl.K;
            a.nb = (int)round_up(std::min(B, 256), 16);
            a.out_f32 = 1;
            a.relu = 0;
            a.out = c->logits;
            a.ldo = c->O;
            a.out_stride_s = (int64_t)B * c->O;
            a.vec_ok = (sl.K % 4 == 0 && sl.off_w % 4 == 0) ? 1 : 0;
            c->launch("fwd", [&] { launch_gen_gemm(c->map_fwdB[0], a, Sc, st); });
            continue;
        }
        const LayerDesc& Ld = c->layers[op.layer];
        const RBuf& Sb = c->rbufs[op.src];
        const RBuf& Db = c->rbufs[op.dst];
        const int Cp = c->rbf[op.src].C_pad;
        if (ahead) cudaStreamWaitEvent(st, c->wgen_ev[op.layer], 0);
        Conv2Args a{};
        a.S = Sc;
        a.B = B;
        a.H = Sb.H;
        a.W = Sb.W;
        a.C = Sb.C;
        a.C_pad = Cp;
        a.OH = Db.H;
        a.OW = Db.W;
        a.CO = Db.C;
        a.k = Ld.k;
        a.stride = Ld.stride;
        a.pad = Ld.pad;
        a.K_pad = c->kpad[op.layer];
        a.n_tile = std::min(Db.C, 256);
        a.tma_a = c->tma_a2f[op.layer];
        a.src = c->rbf[op.src].val;
        a.src_stride_s = op.src == 0 ? in_stride : (int64_t)B * Sb.H * Sb.W * Cp;
        a.out = c->rbf[op.dst].val;
        a.out_stride_s = (int64_t)B * Db.H * Db.W * Db.C;
        a.bias = c->bias_scr + (size_t)op.layer * Sc * 512;
        a.res = op.res >= 0 ? c->rbf[op.res].val : nullptr;
        a.relu = op.relu;
        a.mbits_out = op.relu ? c->rbf[op.dst].mbits : nullptr;
        if (op.layer == c->stem_layer && (a.wsrc = c->wscr + c->wscr_off[op.layer], stem_fwd_ok(a))) {
            c->launch("fwd", [&] { launch_stem_fwd(c->cmap_stem, a, st); });  // two taps per MMA, pixels on M
        } else if (Db.C <= 128) {  // channels on M, 256 pixels on N (full-width MMA)
            a.tma_a = c->tma_fwd[op.layer];
            a.halo = c->halo_fwd[op.layer];
            const CUtensorMap& bm = a.halo ? c->cmap_hf[op.layer] : c->cmap_bf[op.layer];
            if (a.halo && c->conv64[op.layer])
                c->launch("fwd", [&] { launch_conv64_fwd(c->cmap_w64[op.layer], c->rowmaps[op.layer], a, st); });
            else
                c->launch("fwd", [&] { launch_conv3_fwd(Db.C >= 128 ? c->cmap_w[op.layer] : c->cmap_w64[op.layer], bm, a, st); });
        } else {
            c->launch("fwd", [&] { launch_conv2_fwd(c->cmap_a2f[op.layer], c->cmap_w2[op.layer], a, st); });
        }
    }
}

int resnet_bf16_chunk(bnn_ctx* c, const float* mu, const float* x, const int32_t* ycls,
                      const float* yreg, int B, int B_glob, int S_glob, int Sc, uint32_t s0,
                      uint64_t seed, uint32_t step, float* acc_mu, float* acc_rho, float* acc_loss,
                      int phase, bool skip_fwd, const float* gstats) {
    NvtxRange nvtx_("bnn.chunk");
    cudaStream_t st = c->st;
    SampleKeys kk{make_key(seed), step, s0};
    const float scale = c->model.loss == BNN_LOSS_CE ? 1.0f / ((float)S_glob * B_glob)
                                                     : 1.0f / ((float)S_glob * B_glob * c->O);
    const bool aug = c->cfg.aug == BNN_AUG_PER_SAMPLE;
    if (!skip_fwd) {
        NvtxRange nv("bnn.forward");
        resnet_bf16_forward(c, mu, x, Sc, B, seed, step, s0, aug);
    }
    NvtxRange nvb("bnn.backward");
    const RBuf& in = c->rbufs[0];
    const int64_t in_stride = aug ? (int64_t)B * in.H * in.W * c->rbf[0].C_pad : 0;
    const int O = c->O, ldO = (int)round_up(O, 8);
    if (phase == kPhaseStats) {
        c->launch("loss", [&] { launch_mean_stats(c->logits, Sc, B, O, c->mkind(), ycls, c->mstats, (int)(s0 - (uint32_t)(c->kidx * (S_glob / c->K))), st); });
        return BNN_OK;
    }
    if (phase == kPhaseMeanBwd)
        c->launch("loss", [&] {
            launch_mean_loss_head(c->logits, Sc, B, O, c->mkind(), ycls, yreg, gstats, S_glob, c->fcG, ldO, true,
                                  c->dz_f32, st);
        });
    else
        c->launch("loss", [&] {
            launch_loss_head(c->logits, Sc, B, O, c->model.loss, ycls, yreg, c->fcG, ldO, true, c->lossrow,
                             c->dz_f32, st);
        });
    // ---------------- head (linear layer on pooled features)
    const ROp& fc = c->rops.back();
    const ROp& gap = c->rops[c->rops.size() - 2];
    const int gbuf = gap.dst, ylast = gap.src;
    {
        SampledLayer sl = sampled(c, fc.layer, mu);
        TcWgradMaps maps;
        maps.g[0] = c->map_wgG[0];
        maps.x[0] = c->map_wgX[0];
        TcWgradArgs w{};
        w.kk = kk;
        w.S = Sc;
        w.B = B;
        w.scale = scale;
        w.acc_mu = acc_mu;
        w.acc_rho = acc_rho;
        w.nlayers = 1;
        w.lay[0].L = sl;
        w.lay[0].mtiles = (sl.N + 127) / 128;
        w.lay[0].ktiles = (sl.K + kWgradTileK - 1) / kWgradTileK;
        w.lay[0].tile_base = 0;
        w.lay[0].b_shared = 0;
        // weight-side work of every layer (wgrad, ε combine, bias) runs on the side stream,
        // overlapping the data-gradient chain on st (fork after its inputs exist; in order on
        // the side stream, so the shared wpart / db_scratch scratch is reused safely)
        cudaStream_t ss = fork_side(c);
        if (phase == kPhaseFull)
            c->launch("loss", [&] { launch_loss_reduce(c->lossrow, Sc * B, scale, acc_loss, ss); });
        c->launch("wgrad", [&] { launch_wgrad_tc(maps, w, ss); });
        cudaStream_t sb = fork_side2(c);  // every bias launch shares db_scratch: one stream
        c->launch("bias", [&] {
            return launch_bias_grad(sl, kk, Sc, c->dz_f32, B, O, (int64_t)B * O, scale, c->db_scratch, acc_mu, acc_rho, sb);
        });
        TcGenArgs a{};
        a.L = sl;
        a.kk = kk;
        a.mode = 1;
        a.B = B;
        a.M = sl.K;
        a.R = sl.N;
        a.nb = (int)round_up(std::min(B, 256), 16);
        a.out = c->rbf[gbuf].grad;
        a.ldo = sl.K;
        a.out_stride_s = (int64_t)B * sl.K;
        a.mask = nullptr;
        a.dbpart = nullptr;
        a.vec_ok = (sl.K % 4 == 0 && sl.off_w % 4 == 0) ? 1 : 0;
        c->launch("dgrad", [&] { launch_gen_gemm(c->map_dgradB[0], a, Sc, st); });
        int rc = ar_layer_done(c, fc.layer, ss, sb);  // the head's acc segments: bucket candidate
        if (rc) return rc;
    }
    // ---------------- GAP backward (+ ReLU mask of the last block output, bias partials)
    {
        const RBuf& Y = c->rbufs[ylast];
        c->launch("gap", [&] {
            launch_gap_bwd_bf16(c->rbf[gbuf].grad, Y.C, c->rbf[ylast].val, Sc * B, Y.H * Y.W, Y.C,
                                c->rbf[ylast].grad, c->rbf[ylast].bpart, st);
        });
        c->rbf[ylast].nparts = B;
    }
    // ---------------- convolutions in reverse
    const int nb = (int)c->rbufs.size();
    std::vector<int> remaining(nb, 0);
    std::vector<const __nv_bfloat16*> pending(nb, nullptr);
    for (const ROp& op : c->rops) {
        if (op.type != 0 || is_fc(c, op)) continue;
        if (op.src != 0) remaining[op.src]++;
        if (op.res >= 0 && !is_proj_output(c, op.res)) remaining[op.res]++;
    }
    int wbuf = 0;  // wpart buffer of the next conv wgrad (alternates per layer)
    const bool split3 = !c->prof && c->side3;
    for (int oi = (int)c->rops.size() - 1; oi >= 0; --oi) {
        const ROp& op = c->rops[oi];
        if (op.type != 0 || is_fc(c, op)) continue;
        const LayerDesc& Ld = c->layers[op.layer];
        SampledLayer sl = sampled(c, op.layer, mu);
        const int gb = grad_src_buffer(c, op.dst);
        const RBuf& Db = c->rbufs[op.dst];
        const RBuf& Sb = c->rbufs[op.src];
        const bnn_ctx::RBf& G = c->rbf[gb];
        const int64_t npix_out = (int64_t)B * Db.H * Db.W;
        // bias gradient from the fused partials of dL/dz (second side stream: the bias chain
        // and the wgrad / ε-combine chain each overlap the data-gradient chain on st)
        cudaStream_t sb = fork_side2(c);
        c->launch("bias", [&] {
            // many partials (the stage-1 dgrad tiles): 64-part chunks summed in parallel first
            return launch_bias_grad_rows(sl, kk, Sc, G.bpart, G.nparts, Db.C, (int64_t)G.nparts * Db.C, scale,
                                         c->bias_rows_scr, c->bias_rows_cap, c->db_scratch,
                             acc_mu, acc_rho, sb);
        });
        cudaStream_t ss = fork_side(c);
        // weight gradient with the sample-accumulating ε epilogue
        if (Ld.cin % 64 == 0 || c->rbf[op.src].C_pad == 8) {
            ConvWgradArgs w{};
            w.L = sl;
            w.kk = kk;
            w.S = Sc;
            w.B = B;
            w.H = Sb.H;
            w.W = Sb.W;
            w.C = Sb.C;
            w.C_pad = c->rbf[op.src].C_pad;
            w.OH = Db.H;
            w.OW = Db.W;
            w.CO = Db.C;
            w.k = Ld.k;
            w.stride = Ld.stride;
            w.pad = Ld.pad;
            w.X = c->rbf[op.src].val;
            w.X_stride_s = op.src == 0 ? in_stride : (int64_t)B * Sb.H * Sb.W * Sb.C;
            w.scale = scale;
            float* wp = wbuf ? c->wpart2 : c->wpart;
            w.part = wp;
            w.nsplit = c->nsplit[op.layer];
            w.tma_b = c->tma_wgrad[op.layer];
            const int taps = Ld.k * Ld.k, Kt = conv2_wgrad_cols(taps, Ld.cin, w.C_pad);
            w.n_tile = conv2_wgrad_ntile(Kt);
            w.kpx = w.tma_b ? c->wkpx[op.layer] : 64;
            w.cps = c->wcps[op.layer];
            if (w.kpx != c->wkpx[op.layer]) return c->set_err(BNN_ERR_CONFIG, "wgrad k-step / operand path mismatch");
            // the buffer is free once the ε combine that last read it (two layers back) is done
            if (split3) cudaStreamWaitEvent(ss, c->ev_comb[wbuf], 0);
            const bool epsf = c->wgrad_eps[op.layer] && c->conv64[op.layer];
            if (epsf) {  // ε and the sample sum in the GEMM's epilogue (clusters), then the ordered split sum
                w.eps_cluster = conv64_wgrad_eps_cluster(Sc);
                w.nsplit = c->nsplit[op.layer] * (Sc / w.eps_cluster);  // partials: pixel splits × sample groups
                int lrc = 0;
                c->launch("wgrad", [&] { lrc = launch_conv64_wgrad_eps(c->rowmaps[op.layer], w, ss); });
                if (lrc) return c->set_err(BNN_ERR_CUDA, "cluster launch of the ε-fused weight gradient refused");
            } else if (c->conv64[op.layer] && conv64w_layer(c, op))  // both halo window maps exist for conv64 layers
                c->launch("wgrad", [&] { launch_conv64_wgrad(c->rowmaps[op.layer], w, ss); });
            else
                c->launch("wgrad", [&] { launch_conv2_wgrad(c->cmap_g[op.layer], c->cmap_xw[op.layer], w, ss); });
            cudaStream_t sc = ss;
            if (split3) {  // ε combine on the third stream, overlapping the next layer's wgrad GEMM
                cudaEventRecord(c->ev_wg[wbuf], ss);
                cudaStreamWaitEvent(c->side3, c->ev_wg[wbuf], 0);
                sc = c->side3;
            }
            if (epsf) {
                c->launch("wgrad", [&] {
                    launch_wgrad_split_reduce(wp, w.nsplit, (int64_t)Ld.cout * Kt, Ld.off_w, acc_mu, acc_rho, sc);
                });
            } else if (w.C_pad < 64) {
                c->launch("wcomb", [&] {
                    launch_wgrad_eps_combine_stem(sl, kk, Sc, w.nsplit, Ld.cout, taps, Ld.cin, Kt, wp, scale,
                                                  acc_mu, acc_rho, sc);
                });
            } else {
                c->launch("wcomb", [&] {
                    launch_wgrad_eps_combine(sl, kk, Sc, w.nsplit, Ld.cout, Kt, wp, scale, acc_mu, acc_rho, sc);
                });
            }
            if (split3) cudaEventRecord(c->ev_comb[wbuf], sc);
            wbuf ^= 1;
            int rc = ar_layer_done(c, op.layer, sc, sb);  // acc_μ/acc_ρ of this layer final (last chunk)
            if (rc) return rc;
        } else {
            ConvShape cs{B, Sb.H, Sb.W, Sb.C, Db.H, Db.W, Db.C, Ld.k, Ld.stride, Ld.pad};
            const int nsp = c->nsplit[op.layer];
            float* wp = wbuf ? c->wpart2 : c->wpart;
            if (split3) cudaStreamWaitEvent(ss, c->ev_comb[wbuf], 0);
            c->launch("wgrad", [&] {
                launch_conv_wgrad_simt_bf16(sl, kk, Sc, cs, c->rbf[op.src].C_pad, G.grad, npix_out * Db.C,
                                            c->rbf[op.src].val, op.src == 0 ? in_stride : 0, scale, wp,
                                            nsp, ss);
            });
            const int64_t n = (int64_t)Ld.cout * Ld.k * Ld.k * Ld.cin;
            c->launch("wgrad", [&] { launch_wgrad_split_reduce(wp, nsp, n, Ld.off_w, acc_mu, acc_rho, ss); });
            if (split3) cudaEventRecord(c->ev_comb[wbuf], ss);
            wbuf ^= 1;
            int rc = ar_layer_done(c, op.layer, ss, sb);
            if (rc) return rc;
        }
        // identity residual: dL/dy flows unchanged into the block input
        if (op.res >= 0 && !is_proj_output(c, op.res)) {
            remaining[op.res]--;
            pending[op.res] = G.grad;
        }
        if (op.src == 0) continue;
        // data gradient: the transposed implicit GEMM on the forward's W_s slot of this layer
        remaining[op.src]--;
        const bool final = remaining[op.src] == 0;
        Conv2Args a{};
        a.S = Sc;
        a.B = B;
        a.H = Sb.H;
        a.W = Sb.W;
        a.C = Sb.C;
        a.C_pad = c->rbf[op.src].C_pad;
        a.OH = Db.H;
        a.OW = Db.W;
        a.CO = Db.C;
        a.k = Ld.k;
        a.stride = Ld.stride;
        a.pad = Ld.pad;
        a.K_pad = c->kpad[op.layer];
        a.n_tile = std::min(Sb.C, 256);
        a.tma_a = c->tma_a2d[op.layer];
        a.src = G.grad;
        a.src_stride_s = npix_out * Db.C;
        a.out = c->rbf[op.src].grad;
        a.out_stride_s = (int64_t)B * Sb.H * Sb.W * Sb.C;
        const bool m_chan = Sb.C <= 128;  // conv3: channels on M, 256 pixels on N
        if (m_chan) a.tma_a = c->tma_dgrad[op.layer];
        if (m_chan) a.halo = c->halo_dgrad[op.layer];
        if (final) {
            const int np = (m_chan && a.halo && c->conv64[op.layer]) ? conv64_parts(a)
                           : m_chan ? conv3_dgrad_parts(a) : conv2_dgrad_parts(a);
            a.addsrc = pending[op.src];
            a.mbits = c->rbf[op.src].mbits;  // written by the producer's forward epilogue
            a.mask = a.mbits ? nullptr : c->rbf[op.src].val;
            if (!a.mbits && Sb.C <= 128)
                return c->set_err(BNN_ERR_CONFIG, "conv3 dgrad needs the ReLU bitmask of its input");
            a.bpart = c->rbf[op.src].bpart;
            a.bpart_stride_s = (int64_t)np * Sb.C;
            if ((int64_t)np * Sb.C > c->rbf[op.src].bpart_cap)
                return c->set_err(BNN_ERR_CONFIG, "bias partial buffer too small");
            c->rbf[op.src].nparts = np;
        }
        if (m_chan) {
            const CUtensorMap& bm = a.halo ? c->cmap_hd[op.layer] : c->cmap_bd[op.layer];
            if (a.halo && c->conv64[op.layer])
                c->launch("dgrad", [&] { launch_conv64_dgrad(c->cmap_wT[op.layer], c->rowmaps[op.layer], a, st); });
            else
                c->launch("dgrad", [&] { launch_conv3_dgrad(c->cmap_wT[op.layer], bm, a, st); });
        } else {
            c->launch("dgrad", [&] { launch_conv2_dgrad(c->cmap_a2d[op.layer], c->cmap_wT[op.layer], a, st); });
        }
        if (!final) pending[op.src] = c->rbf[op.src].grad;
    }
    join_side(c);  // the next chunk's forward overwrites what the side stream reads
    return BNN_OK;
}
