/*
 * bnn_oracle.c — the CPU oracle for the Bayes-by-backprop ELBO step.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the slow, plain, obviously-correct reference
 * that the CUDA path is checked against. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product path
 * (paper_2604_04736_b200/) never links, imports or executes it, and it shares no code,
 * header, constant table or helper with the CUDA path.
 *
 * Arithmetic is IEEE binary64 throughout, except ε, which is produced as binary32 bits
 * by EPS-v1 (docs/EPS.md) and widened to double.
 *
 * What it computes:
 *   Alg. 1 (§2.1) applied to one minibatch; Alg. 2 (PAPER.md:250-265,
 *   §4.1) yields the same value for any sharding of samples/examples.
 *     σ = softplus(ρ)                                      (reading R1)
 *     ε_s ~ N(0, I) via EPS-v1                              (Alg.1 l.5)
 *     w_s = μ + σ ⊙ ε_s                                     (Alg.1 l.6)
 *     ŷ_s = ForwardPass(x, w_s)                             (Alg.1 l.7)
 *     L_data = (1/S) Σ_s Loss(ŷ_s, y)                       (Alg.1 l.9)
 *     L_KL   = ½ Σ_i (σ_i² + μ_i² − 1 − log σ_i²)           (Alg.1 l.10)
 *     L      = L_data + L_KL / |D|                           (Alg.1 l.11)
 *     ∇L(μ, σ) by the chain rule, mapped to ρ via dσ/dρ = sigmoid(ρ)
 *   Loss(ŷ_s, y) is the batch mean of per-example cross-entropy (or of squared error over
 *   batch×outputs) — DESIGN.md readings R5-R7.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py and
 * tests/test_eps_oracle.py (closed forms, finite differences, torch-autograd cross-check,
 * brute force, Random123 known answers, exhaustive libm sweeps). Full-size C2-C5 values
 * are "parity unpinned" beyond those structural pins.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC (see oracle/build.sh)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if defined(__FAST_MATH__)
#error "oracle must be built without fast-math"
#endif

/* ======================================================================================
 * Part 1. EPS-v1 (docs/EPS.md). Written from the spec; independent of the CUDA copy.
 * ====================================================================================== */

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* Philox4x32-10 (docs/EPS.md §2). */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t x0 = ctr_in[0], x1 = ctr_in[1], x2 = ctr_in[2], x3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ x1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ x3 ^ k1;
        uint32_t n3 = lo0;
        x0 = n0; x1 = n1; x2 = n2; x3 = n3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* LOG24 (docs/EPS.md §3): u must be k·2^-24, k in [1, 2^24]. */
float orc_log24(float u)
{
    const float Q0 = -0x1.fffffap-2f, Q1 = 0x1.5556f4p-2f, Q2 = -0x1.00049ap-2f,
                Q3 = 0x1.98d2bap-3f, Q4 = -0x1.535d4cp-3f, Q5 = 0x1.31857cp-3f,
                Q6 = -0x1.2503eap-3f, Q7 = 0x1.65c3bap-4f;
    const float LN2_HI = 0x1.62e4p-1f, LN2_LO = 0x1.7f7d1cp-20f;
    uint32_t ix = f2u(u) - 0x3F3504F3u;
    int32_t e = ((int32_t)ix) >> 23;
    float m = u2f((ix & 0x007FFFFFu) + 0x3F3504F3u);
    float f = m - 1.0f;
    float q = Q7;
    q = fmaf(q, f, Q6);
    q = fmaf(q, f, Q5);
    q = fmaf(q, f, Q4);
    q = fmaf(q, f, Q3);
    q = fmaf(q, f, Q2);
    q = fmaf(q, f, Q1);
    q = fmaf(q, f, Q0);
    float f2 = f * f;
    float y = fmaf(f2, q, f);
    float ef = (float)e;
    return fmaf(ef, LN2_HI, fmaf(ef, LN2_LO, y));
}

/* SINCOS2PI24 (docs/EPS.md §3): v is a 24-bit angle index. */
void orc_sincos2pi24(uint32_t v, float* cos_out, float* sin_out)
{
    const float S0 = 0x1.921fb6p-1f, S1 = -0x1.4abbbap-4f, S2 = 0x1.465e94p-9f,
                S3 = -0x1.2d9368p-15f;
    const float C0 = 0x1p+0f, C1 = -0x1.3bd3ccp-2f, C2 = 0x1.03c1dap-6f,
                C3 = -0x1.55c4ecp-12f, C4 = 0x1.d99fbep-19f;
    uint32_t w = (v + 0x200000u) & 0xFFFFFFu;
    uint32_t q = w >> 22;
    float t = (float)((int32_t)(w & 0x3FFFFFu) - 0x200000) * 0x1p-21f;
    float t2 = t * t;
    float ps = fmaf(t2, S3, S2);
    ps = fmaf(t2, ps, S1);
    ps = fmaf(t2, ps, S0);
    float s = t * ps;
    float pc = fmaf(t2, C4, C3);
    pc = fmaf(t2, pc, C2);
    pc = fmaf(t2, pc, C1);
    float c = fmaf(t2, pc, C0);
    float C, S;
    switch (q) {
        case 0: C = c; S = s; break;
        case 1: C = -s; S = c; break;
        case 2: C = -c; S = -s; break;
        default: C = s; S = -c; break;
    }
    *cos_out = C;
    *sin_out = S;
}

/* ε for (seed, step, global sample s, tensor t, row r, column c) — docs/EPS.md §1-3. */
float orc_eps(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r, uint32_t c)
{
    uint32_t ctr[4] = {c >> 2, r, (t << 20) | s, step};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t y[4];
    orc_philox4x32_10(ctr, key, y);
    uint32_t j = c & 3u;
    uint32_t a = (j < 2) ? y[0] : y[2];
    uint32_t b = (j < 2) ? y[1] : y[3];
    float u = (float)((a >> 8) + 1u) * 0x1p-24f;
    float L = orc_log24(u);
    float R = sqrtf(L * -2.0f);
    float C, S;
    orc_sincos2pi24(b >> 8, &C, &S);
    return (j % 2 == 0) ? R * C : R * S;
}

/* Fill out[i*nc + k] = ε(seed, step, s, t, r0+i, c0+k). */
void orc_eps_fill(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r0,
                  uint32_t nr, uint32_t c0, uint32_t nc, float* out)
{
    #pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)nr; ++i)
        for (uint32_t k = 0; k < nc; ++k)
            out[(size_t)i * nc + k] = orc_eps(seed, step, s, t, r0 + (uint32_t)i, c0 + k);
}

/* Augmentation parameters (docs/EPS.md §4). */
void orc_aug_params(uint64_t seed, uint32_t step, uint32_t s, uint32_t b, int* dx, int* dy,
                    int* flip)
{
    uint32_t ctr[4] = {0u, b, (4095u << 20) | s, step};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t y[4];
    orc_philox4x32_10(ctr, key, y);
    *dx = (int)(y[0] % 9u);
    *dy = (int)(y[1] % 9u);
    *flip = (int)(y[2] & 1u);
}

/* MC-dropout mask (R25): unit j of hidden layer
 * `layer` for global example b under sample s is kept iff the 24 high bits of Philox word
 * (b & 3) of counter ((layer << 24) | (b >> 2), j, (4094 << 20) | s, step) are ≥ P24, the drop
 * probability in units of 2^-24 (P24 = round(p·2^24)). Integer decision: bit-exact everywhere. */
int orc_dropout_keep(uint64_t seed, uint32_t step, uint32_t s, uint32_t layer, uint32_t b, uint32_t j,
                     uint32_t p24)
{
    uint32_t ctr[4] = {(layer << 24) | (b >> 2), j, (4094u << 20) | s, step};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t y[4];
    orc_philox4x32_10(ctr, key, y);
    return (y[b & 3u] >> 8) >= p24;
}

/* ======================================================================================
 * Part 2. The model: every layer is a convolution over an NHWC image (a linear layer is
 * a 1×1 convolution over a 1×1 image). Tensor layout: for each layer in
 * model order, weight t = 2l viewed as [rows = c_out, cols = kh·kw·c_in] (OHWI, c_in
 * fastest), then bias t = 2l+1 viewed as [1, c_out].
 * ====================================================================================== */

enum { ORC_MLP = 0, ORC_RESNET18 = 1 };
enum { ORC_CE = 0, ORC_MSE = 1, ORC_GNLL = 2 /* mean-prediction aggregation only */ };
/* variance floor of the Gaussian NLL of the predictive distribution (reading R24) */
#define ORC_GNLL_EPS 1e-6
#define ORC_TWO_PI 6.283185307179586476925286766559
enum { ORC_RELU = 0, ORC_TANH = 1 };
enum { ORC_AUG_NONE = 0, ORC_AUG_PER_SAMPLE = 1 };

/* The oracle's own model description (field meanings documented in DESIGN.md §3). */
typedef struct {
    int kind;        /* ORC_MLP | ORC_RESNET18 */
    int n_widths;    /* MLP: number of entries in widths (layers = n_widths-1) */
    int widths[16];  /* MLP: widths[0] = input features, widths[n-1] = outputs */
    int in_h, in_w, in_c, n_classes; /* ResNet-18 input image and classes */
    int base_width;  /* ResNet-18 stage-1 width (64 for the paper-shaped model) */
    int loss;        /* ORC_CE | ORC_MSE | ORC_GNLL */
    int act;         /* ORC_RELU (the model) | ORC_TANH (FD self-check variant only) */
    int mcd;         /* 1: MC dropout (f4): weights μ, dropout after every hidden activation */
    double dropout_p;
} orc_model;

typedef struct { int cin, cout, k, stride, pad; long off_w, off_b; } OLayer;

enum { OP_CONV = 0, OP_ACT = 1, OP_ADD = 2, OP_GAP = 3 };
typedef struct { int type, layer, src, dst; } OOp;

#define MAXL 64
#define MAXOPS 160
#define MAXBUF 96

typedef struct {
    int n_layers, n_ops, n_bufs;
    OLayer L[MAXL];
    OOp ops[MAXOPS];
    int bh[MAXBUF], bw[MAXBUF], bc[MAXBUF]; /* buffer shapes (H, W, C) */
    long n_params;
    int n_out, loss, act;
    int mcd;            /* MC dropout (R25) */
    uint32_t p24;       /* drop threshold, units of 2^-24 */
    double inv_keep;    /* 1 / (1 − p) */
    int in_h, in_w, in_c;
    int has_act[MAXBUF];   /* an activation is applied to the buffer (BF16 emulation) */
    int n_contrib[MAXBUF]; /* backward contributions to the buffer's gradient */
    int out_buf;
} ONet;

static int add_buf(ONet* n, int h, int w, int c)
{
    n->bh[n->n_bufs] = h; n->bw[n->n_bufs] = w; n->bc[n->n_bufs] = c;
    return n->n_bufs++;
}
static int add_layer(ONet* n, int cin, int cout, int k, int stride, int pad)
{
    OLayer* L = &n->L[n->n_layers];
    L->cin = cin; L->cout = cout; L->k = k; L->stride = stride; L->pad = pad;
    L->off_w = n->n_params; n->n_params += (long)cout * k * k * cin;
    L->off_b = n->n_params; n->n_params += cout;
    return n->n_layers++;
}
static void add_op(ONet* n, int type, int layer, int src, int dst)
{
    OOp* o = &n->ops[n->n_ops++];
    o->type = type; o->layer = layer; o->src = src; o->dst = dst;
}
static int conv_out(int x, int k, int s, int p) { return (x + 2 * p - k) / s + 1; }

/* conv + (optional) act, returns dst buffer */
static int emit_conv(ONet* n, int src, int cout, int k, int stride, int pad, int act)
{
    int h = conv_out(n->bh[src], k, stride, pad), w = conv_out(n->bw[src], k, stride, pad);
    int l = add_layer(n, n->bc[src], cout, k, stride, pad);
    int dst = add_buf(n, h, w, cout);
    add_op(n, OP_CONV, l, src, dst);
    if (act) add_op(n, OP_ACT, -1, dst, dst);
    return dst;
}

static int build_net_(const orc_model* m, ONet* n);
static void net_flags(ONet* n);
static int build_net(const orc_model* m, ONet* n)
{
    int rc = build_net_(m, n);
    if (!rc) net_flags(n);
    return rc;
}
static int build_net_(const orc_model* m, ONet* n)
{
    memset(n, 0, sizeof(*n));
    n->loss = m->loss; n->act = m->act;
    n->mcd = m->mcd;
    if (m->mcd) {
        if (m->kind != ORC_MLP || m->act != ORC_RELU || !(m->dropout_p >= 0.0 && m->dropout_p < 1.0)) return -1;
        n->p24 = (uint32_t)llround(m->dropout_p * 16777216.0);
        n->inv_keep = 1.0 / (1.0 - m->dropout_p);
    }
    if (m->kind == ORC_MLP) {
        if (m->n_widths < 2 || m->n_widths > 16) return -1;
        n->in_h = 1; n->in_w = 1; n->in_c = m->widths[0];
        int cur = add_buf(n, 1, 1, m->widths[0]);
        for (int i = 1; i < m->n_widths; ++i)
            cur = emit_conv(n, cur, m->widths[i], 1, 1, 0, i < m->n_widths - 1);
        n->n_out = m->widths[m->n_widths - 1];
        return 0;
    }
    if (m->kind == ORC_RESNET18) {
        /* CIFAR ResNet-18 topology without BatchNorm (reading R12). */
        n->in_h = m->in_h; n->in_w = m->in_w; n->in_c = m->in_c;
        int bw0 = m->base_width > 0 ? m->base_width : 64;
        int cur = add_buf(n, m->in_h, m->in_w, m->in_c);
        cur = emit_conv(n, cur, bw0, 3, 1, 1, 1); /* stem */
        int width = bw0;
        for (int stage = 0; stage < 4; ++stage) {
            int cout = bw0 << stage;
            for (int blk = 0; blk < 2; ++blk) {
                int stride = (stage > 0 && blk == 0) ? 2 : 1;
                int in = cur;
                int a = emit_conv(n, in, cout, 3, stride, 1, 1);      /* conv1 + act */
                int b = emit_conv(n, a, cout, 3, 1, 1, 0);            /* conv2 */
                if (stride != 1 || width != cout) {
                    int sc = emit_conv(n, in, cout, 1, stride, 0, 0);  /* 1×1 projection */
                    add_op(n, OP_ADD, -1, sc, b);
                } else {
                    add_op(n, OP_ADD, -1, in, b);
                }
                add_op(n, OP_ACT, -1, b, b);
                cur = b;
                width = cout;
            }
        }
        int g = add_buf(n, 1, 1, width);
        add_op(n, OP_GAP, -1, cur, g);
        emit_conv(n, g, m->n_classes, 1, 1, 0, 0); /* FC */
        n->n_out = m->n_classes;
        return 0;
    }
    return -1;
}

static void net_flags(ONet* n)
{
    for (int b = 0; b < MAXBUF; ++b) { n->has_act[b] = 0; n->n_contrib[b] = 0; }
    for (int i = 0; i < n->n_ops; ++i) {
        const OOp* o = &n->ops[i];
        if (o->type == OP_ACT) n->has_act[o->dst] = 1;
        if (o->type == OP_CONV || o->type == OP_ADD || o->type == OP_GAP)
            if (o->src != 0) n->n_contrib[o->src]++;
        if (o->type == OP_CONV || o->type == OP_GAP) n->out_buf = o->dst;
    }
}

long orc_n_params(const orc_model* m)
{
    ONet n;
    if (build_net(m, &n)) return -1;
    return n.n_params;
}
int orc_n_tensors(const orc_model* m)
{
    ONet n;
    if (build_net(m, &n)) return -1;
    return 2 * n.n_layers;
}
/* info = {offset, rows, cols, kh, cin, stride, pad} for tensor t. */
int orc_tensor_info(const orc_model* m, int t, long* info)
{
    ONet n;
    if (build_net(m, &n) || t < 0 || t >= 2 * n.n_layers) return -1;
    const OLayer* L = &n.L[t / 2];
    if (t % 2 == 0) {
        info[0] = L->off_w; info[1] = L->cout; info[2] = (long)L->k * L->k * L->cin;
    } else {
        info[0] = L->off_b; info[1] = 1; info[2] = L->cout;
    }
    info[3] = L->k; info[4] = L->cin; info[5] = L->stride; info[6] = L->pad;
    return 0;
}

/* ---------------------------------------------------------------------------------- */
static double softplus(double r) { return (r > 0 ? r : 0.0) + log1p(exp(-fabs(r))); }
static double sigmoid(double r)
{
    if (r >= 0) return 1.0 / (1.0 + exp(-r));
    double e = exp(r);
    return e / (1.0 + e);
}
/* ln(softplus(ρ)), accurate also for very negative ρ (reading R4). */
static double log_softplus(double r)
{
    if (r < -30.0) return r + log1p(-0.5 * exp(r)); /* softplus(ρ) = e^ρ(1 − e^ρ/2 + …) */
    return log(softplus(r));
}

/* ---- BF16 emulation (reading R14): the rounding points of the BF16 tensor-core
 * mode, written from that reading (not from the CUDA code): w_s = RN_bf16(fma_f32(σ, ε, μ)),
 * biases fma_f32; the network input and every stored activation RN_bf16 (logits stay fp32);
 * gradients RN_bf16 where they are stored between layers, with the bias gradient taken from
 * the unrounded value; accumulation in (here: double) precision. */
static double bf16r(double x)
{
    float f = (float)x;
    uint32_t u;
    memcpy(&u, &f, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u; /* round to nearest even */
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Sampled weights for global sample s: W = μ + σ·ε. eps_out optional. */
static void sample_weights(const ONet* n, const double* mu, const double* sigma,
                           uint64_t seed, uint32_t step, uint32_t s, double* W, double* eps_out,
                           int emu)
{
    if (n->mcd) {  /* MC dropout (R25): deterministic weights μ; the BF16 operand is RN_bf16(μ) */
        for (long i = 0; i < n->n_params; ++i) {
            W[i] = mu[i];
            if (eps_out) eps_out[i] = 0.0;
        }
        if (emu)
            for (int l = 0; l < n->n_layers; ++l) {
                const OLayer* L = &n->L[l];
                long nw = (long)L->cout * L->k * L->k * L->cin;
                for (long i = 0; i < nw; ++i) W[L->off_w + i] = bf16r((double)(float)mu[L->off_w + i]);
            }
        return;
    }
    for (int l = 0; l < n->n_layers; ++l) {
        const OLayer* L = &n->L[l];
        long cols = (long)L->k * L->k * L->cin;
        for (int r = 0; r < L->cout; ++r)
            for (long c = 0; c < cols; ++c) {
                long i = L->off_w + r * cols + c;
                double e = (double)orc_eps(seed, step, s, (uint32_t)(2 * l), (uint32_t)r,
                                           (uint32_t)c);
                W[i] = emu ? bf16r(fmaf((float)sigma[i], (float)e, (float)mu[i]))
                           : mu[i] + sigma[i] * e;
                if (eps_out) eps_out[i] = e;
            }
        for (int c = 0; c < L->cout; ++c) {
            long i = L->off_b + c;
            double e = (double)orc_eps(seed, step, s, (uint32_t)(2 * l + 1), 0u, (uint32_t)c);
            W[i] = emu ? (double)fmaf((float)sigma[i], (float)e, (float)mu[i]) : mu[i] + sigma[i] * e;
            if (eps_out) eps_out[i] = e;
        }
    }
}

/* y[oh,ow,co] = b[co] + Σ x[oh·s+kh−p, ow·s+kw−p, ci] · W[co,kh,kw,ci] */
static void conv_fwd(const OLayer* L, const double* W, const double* x, int H, int Wd,
                     double* y, int OH, int OW)
{
    const double* w = W + L->off_w;
    const double* b = W + L->off_b;
    int K = L->k, C = L->cin;
    for (int oh = 0; oh < OH; ++oh)
        for (int ow = 0; ow < OW; ++ow)
            for (int co = 0; co < L->cout; ++co) {
                double acc = b[co];
                for (int kh = 0; kh < K; ++kh) {
                    int ih = oh * L->stride + kh - L->pad;
                    if (ih < 0 || ih >= H) continue;
                    for (int kw = 0; kw < K; ++kw) {
                        int iw = ow * L->stride + kw - L->pad;
                        if (iw < 0 || iw >= Wd) continue;
                        const double* xp = x + ((long)ih * Wd + iw) * C;
                        const double* wp = w + (((long)co * K + kh) * K + kw) * C;
                        for (int ci = 0; ci < C; ++ci) acc += xp[ci] * wp[ci];
                    }
                }
                y[((long)oh * OW + ow) * L->cout + co] = acc;
            }
}

/* dW += scale·g ⊗ x (per the conv's index map), db += scale·Σ g, gx += convᵀ(g) (gx may be
 * NULL). With emu the weight and data gradients use RN_bf16(g), the bias the unrounded g. */
static void conv_bwd(const OLayer* L, const double* W, const double* x, int H, int Wd,
                     const double* g, int OH, int OW, double* dW, double* gx, double scale,
                     int emu)
{
    const double* w = W + L->off_w;
    double* dw = dW + L->off_w;
    double* db = dW + L->off_b;
    int K = L->k, C = L->cin;
    for (int oh = 0; oh < OH; ++oh)
        for (int ow = 0; ow < OW; ++ow)
            for (int co = 0; co < L->cout; ++co) {
                double gv = g[((long)oh * OW + ow) * L->cout + co];
                db[co] += scale * gv;
                if (emu) gv = bf16r(gv);
                const double sgv = scale * gv;
                for (int kh = 0; kh < K; ++kh) {
                    int ih = oh * L->stride + kh - L->pad;
                    if (ih < 0 || ih >= H) continue;
                    for (int kw = 0; kw < K; ++kw) {
                        int iw = ow * L->stride + kw - L->pad;
                        if (iw < 0 || iw >= Wd) continue;
                        long xo = ((long)ih * Wd + iw) * C;
                        long wo = (((long)co * K + kh) * K + kw) * C;
                        for (int ci = 0; ci < C; ++ci) dw[wo + ci] += sgv * x[xo + ci];
                        if (gx)
                            for (int ci = 0; ci < C; ++ci) gx[xo + ci] += gv * w[wo + ci];
                    }
                }
            }
}

static double act_f(int act, double z) { return act == ORC_TANH ? tanh(z) : (z > 0 ? z : 0.0); }
/* derivative expressed through the activation OUTPUT a (ReLU'(0) = 0, reading R13) */
static double act_d(int act, double a) { return act == ORC_TANH ? 1.0 - a * a : (a > 0 ? 1.0 : 0.0); }

typedef struct {
    double* val[MAXBUF];
    double* grad[MAXBUF];
    double* pool;
    /* MC-dropout mask key of the example being processed (set by drop_ctx before forward_one) */
    uint64_t seed;
    uint32_t step, s, bg;
} OWork;

static void drop_ctx(OWork* w, uint64_t seed, uint32_t step, uint32_t s, int b_global)
{
    w->seed = seed; w->step = step; w->s = s; w->bg = (uint32_t)b_global;
}

/* layer whose convolution writes buffer b (MLP: every hidden activation buffer has one) */
static int producer_layer(const ONet* n, int b)
{
    for (int i = 0; i < n->n_ops; ++i)
        if (n->ops[i].type == OP_CONV && n->ops[i].dst == b) return n->ops[i].layer;
    return -1;
}

static long buf_size(const ONet* n, int b) { return (long)n->bh[b] * n->bw[b] * n->bc[b]; }

static int work_alloc(const ONet* n, OWork* w, int with_grad)
{
    long tot = 0;
    for (int b = 0; b < n->n_bufs; ++b) tot += buf_size(n, b) * (with_grad ? 2 : 1);
    w->pool = (double*)calloc((size_t)tot, sizeof(double));
    if (!w->pool) return -1;
    double* p = w->pool;
    for (int b = 0; b < n->n_bufs; ++b) { w->val[b] = p; p += buf_size(n, b); }
    for (int b = 0; b < n->n_bufs; ++b) {
        if (with_grad) { w->grad[b] = p; p += buf_size(n, b); } else w->grad[b] = NULL;
    }
    return 0;
}

/* Forward one example (buffer 0 must hold the input). Returns the output buffer index. */
static void round_buf(const ONet* n, OWork* w, int b)
{
    long sz = buf_size(n, b);
    for (long k = 0; k < sz; ++k) w->val[b][k] = bf16r(w->val[b][k]);
}

static int forward_one(const ONet* n, const double* W, OWork* w, int emu)
{
    if (emu) round_buf(n, w, 0);
    int last = 0;
    for (int i = 0; i < n->n_ops; ++i) {
        const OOp* o = &n->ops[i];
        switch (o->type) {
            case OP_CONV:
                conv_fwd(&n->L[o->layer], W, w->val[o->src], n->bh[o->src], n->bw[o->src],
                         w->val[o->dst], n->bh[o->dst], n->bw[o->dst]);
                last = o->dst;
                /* a stored conv output without activation (projection) is bf16 too */
                if (emu && !n->has_act[o->dst] && o->dst != n->out_buf) round_buf(n, w, o->dst);
                break;
            case OP_ACT: {
                long sz = buf_size(n, o->dst);
                for (long k = 0; k < sz; ++k) w->val[o->dst][k] = act_f(n->act, w->val[o->dst][k]);
                if (n->mcd) {  /* inverted dropout after the hidden activation (R25) */
                    const int l = producer_layer(n, o->dst);
                    for (long k = 0; k < sz; ++k)
                        w->val[o->dst][k] *= orc_dropout_keep(w->seed, w->step, w->s, (uint32_t)l, w->bg,
                                                              (uint32_t)k, n->p24) ? n->inv_keep : 0.0;
                }
                if (emu) round_buf(n, w, o->dst);
                break;
            }
            case OP_ADD: {
                long sz = buf_size(n, o->dst);
                for (long k = 0; k < sz; ++k) w->val[o->dst][k] += w->val[o->src][k];
                break;
            }
            case OP_GAP: {
                int HW = n->bh[o->src] * n->bw[o->src], C = n->bc[o->src];
                for (int c = 0; c < C; ++c) {
                    double acc = 0.0;
                    for (int p = 0; p < HW; ++p) acc += w->val[o->src][(long)p * C + c];
                    w->val[o->dst][c] = acc / HW;
                }
                if (emu) round_buf(n, w, o->dst);
                last = o->dst;
                break;
            }
        }
    }
    return last;
}

/* Backward one example; grad of the output buffer must be set; accumulates into dW.
 * With emu, a gradient contribution that is stored before it is summed (every contribution
 * to a buffer except the last one in reverse order) is RN_bf16, and GAP's incoming gradient
 * (the stored head dgrad) is RN_bf16. tmp holds one contribution (≥ the largest buffer). */
static void backward_one(const ONet* n, const double* W, OWork* w, double* dW, double scale,
                         int emu, double* tmp)
{
    int seen[MAXBUF] = {0};
    for (int i = n->n_ops - 1; i >= 0; --i) {
        const OOp* o = &n->ops[i];
        switch (o->type) {
            case OP_CONV: {
                if (!emu || o->src == 0) {
                    conv_bwd(&n->L[o->layer], W, w->val[o->src], n->bh[o->src], n->bw[o->src],
                             w->grad[o->dst], n->bh[o->dst], n->bw[o->dst], dW,
                             o->src == 0 ? NULL : w->grad[o->src], scale, emu);
                    break;
                }
                long sz = buf_size(n, o->src);
                memset(tmp, 0, sizeof(double) * (size_t)sz);
                conv_bwd(&n->L[o->layer], W, w->val[o->src], n->bh[o->src], n->bw[o->src],
                         w->grad[o->dst], n->bh[o->dst], n->bw[o->dst], dW, tmp, scale, emu);
                int last = ++seen[o->src] == n->n_contrib[o->src];
                for (long k = 0; k < sz; ++k) w->grad[o->src][k] += last ? tmp[k] : bf16r(tmp[k]);
                break;
            }
            case OP_ACT: {
                long sz = buf_size(n, o->dst);
                /* MC dropout: the stored value is ReLU(z)·m/(1−p), so 1[value > 0] = m·1[z > 0]
                 * and the kept units' gradient carries the 1/(1−p) scale */
                const double f = n->mcd ? n->inv_keep : 1.0;
                for (long k = 0; k < sz; ++k) w->grad[o->dst][k] *= act_d(n->act, w->val[o->dst][k]) * f;
                break;
            }
            case OP_ADD: {
                if (o->src == 0) break;
                long sz = buf_size(n, o->dst);
                int last = ++seen[o->src] == n->n_contrib[o->src];
                int rnd = emu && n->has_act[o->src] && !last;
                for (long k = 0; k < sz; ++k)
                    w->grad[o->src][k] += rnd ? bf16r(w->grad[o->dst][k]) : w->grad[o->dst][k];
                break;
            }
            case OP_GAP: {
                int HW = n->bh[o->src] * n->bw[o->src], C = n->bc[o->src];
                ++seen[o->src];
                for (int p = 0; p < HW; ++p)
                    for (int c = 0; c < C; ++c) {
                        double g = emu ? bf16r(w->grad[o->dst][c]) : w->grad[o->dst][c];
                        w->grad[o->src][(long)p * C + c] += g / HW;
                    }
                break;
            }
        }
    }
}

/* Input of example b (global index) under sample s, with optional PER_SAMPLE augmentation. */
static void load_input(const ONet* n, const double* x, int b_local, int b_global, uint64_t seed,
                       uint32_t step, uint32_t s, int aug, double* dst)
{
    int H = n->in_h, Wd = n->in_w, C = n->in_c;
    const double* src = x + (long)b_local * H * Wd * C;
    if (aug != ORC_AUG_PER_SAMPLE) {
        memcpy(dst, src, sizeof(double) * (size_t)H * Wd * C);
        return;
    }
    int dx, dy, flip;
    orc_aug_params(seed, step, s, (uint32_t)b_global, &dx, &dy, &flip);
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < Wd; ++j) {
            int jj = flip ? Wd - 1 - j : j;
            int si = i + dy - 4, sj = jj + dx - 4;
            for (int c = 0; c < C; ++c)
                dst[((long)i * Wd + j) * C + c] =
                    (si >= 0 && si < H && sj >= 0 && sj < Wd) ? src[((long)si * Wd + sj) * C + c] : 0.0;
        }
}

/* Per-example data loss and the seed gradient dℓ/dz (unscaled). */
static double loss_one(const ONet* n, const double* z, const int* ycls, const double* yreg,
                       int b_local, double* dz)
{
    int O = n->n_out;
    if (n->loss == ORC_CE) {
        double mx = z[0];
        for (int k = 1; k < O; ++k) if (z[k] > mx) mx = z[k];
        double se = 0.0;
        for (int k = 0; k < O; ++k) se += exp(z[k] - mx);
        double lse = mx + log(se);
        int y = ycls[b_local];
        for (int k = 0; k < O; ++k) dz[k] = exp(z[k] - lse) - (k == y ? 1.0 : 0.0);
        return lse - z[y];
    }
    double l = 0.0;
    for (int k = 0; k < O; ++k) {
        double d = z[k] - yreg[(long)b_local * O + k];
        l += d * d;
        dz[k] = 2.0 * d;
    }
    return l;
}

/*
 * Partial ELBO data term for samples [s0, s1) and local examples [0, B_loc) whose global
 * indices are b_offset + b (the shard of one rank in a K×G grid).
 *   acc[0 .. P)   += Σ_s Σ_b dℓ_{s,b}/dw · 1/(S·B_glob)           (→ Σ_s dW_s)
 *   acc[P .. 2P)  += Σ_s ε_s ⊙ (Σ_b dℓ_{s,b}/dw) · 1/(S·B_glob)     (→ Σ_s dW_s ⊙ ε_s)
 *   acc[2P]       += Σ_s Σ_b ℓ_{s,b} / (S·B_glob · (O if MSE))
 * Sums are in a fixed order for a fixed thread count.
 */
static int elbo_partial_core(const orc_model* m, const double* mu, const double* rho,
                             const double* x, const int* ycls, const double* yreg, int B_loc,
                             int b_offset, int B_glob, int S_glob, int s0, int s1, uint64_t seed,
                             uint32_t step, int aug, double* acc, int nthreads, int emu,
                             const double* seeds);

int orc_elbo_partial_ex(const orc_model* m, const double* mu, const double* rho, const double* x,
                        const int* ycls, const double* yreg, int B_loc, int b_offset, int B_glob,
                        int S_glob, int s0, int s1, uint64_t seed, uint32_t step, int aug,
                        double* acc, int nthreads, int emu)
{
    return elbo_partial_core(m, mu, rho, x, ycls, yreg, B_loc, b_offset, B_glob, S_glob, s0, s1,
                             seed, step, aug, acc, nthreads, emu, NULL);
}

/* seeds == NULL: the per-sample loss of loss_one (Alg. 1 l.9). Otherwise seeds[s][b][O]
 * (global sample s, local example b) is the complete ∂L_data/∂z_{s,b}, scale included, and
 * no loss is accumulated (the exact-aggregation step below computes L_data itself). */
static int elbo_partial_core(const orc_model* m, const double* mu, const double* rho,
                             const double* x, const int* ycls, const double* yreg, int B_loc,
                             int b_offset, int B_glob, int S_glob, int s0, int s1, uint64_t seed,
                             uint32_t step, int aug, double* acc, int nthreads, int emu,
                             const double* seeds)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    ONet* n = &net;
    long P = n->n_params;
    /* emu = 1: every R14 rounding point; emu = 2: only the sampled weight of the BF16 mode,
     * w_s = RN_bf16(fma_f32(σ, ε, μ)) (R14's definition of w_s), everything else exact fp64 */
    const int emu_act = emu == 1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    double* sigma = (double*)malloc(sizeof(double) * P);
    double* W = (double*)malloc(sizeof(double) * P);
    double* E = (double*)malloc(sizeof(double) * P);
    double* dWt = (double*)calloc((size_t)P * nthreads, sizeof(double));
    double* lt = (double*)calloc((size_t)nthreads, sizeof(double));
    if (!sigma || !W || !E || !dWt || !lt) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    const double scale = (n->loss == ORC_CE) ? 1.0 / ((double)S_glob * B_glob)
                                             : 1.0 / ((double)S_glob * B_glob * n->n_out);
    OWork* works = (OWork*)calloc((size_t)nthreads, sizeof(OWork));
    if (!works) return -2;
    long maxbuf = 0;
    for (int b = 0; b < n->n_bufs; ++b) if (buf_size(n, b) > maxbuf) maxbuf = buf_size(n, b);
    double* tmps = (double*)malloc(sizeof(double) * (size_t)maxbuf * nthreads);
    if (!tmps) return -2;
    for (int t = 0; t < nthreads; ++t)
        if (work_alloc(n, &works[t], 1)) return -2;
    for (int s = s0; s < s1; ++s) {
        sample_weights(n, mu, sigma, seed, step, (uint32_t)s, W, E, emu);
        memset(dWt, 0, sizeof(double) * (size_t)P * nthreads);
        memset(lt, 0, sizeof(double) * (size_t)nthreads);
        #pragma omp parallel num_threads(nthreads)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            OWork* w = &works[tid];
            double dz[4096];
            #pragma omp for schedule(static)
            for (int b = 0; b < B_loc; ++b) {
                for (int k = 0; k < n->n_bufs; ++k)
                    memset(w->grad[k], 0, sizeof(double) * (size_t)buf_size(n, k));
                load_input(n, x, b, b_offset + b, seed, step, (uint32_t)s, aug, w->val[0]);
                drop_ctx(w, seed, step, (uint32_t)s, b_offset + b);
                int out = forward_one(n, W, w, emu_act);
                if (seeds) {
                    const double* sd = seeds + ((size_t)s * B_loc + b) * n->n_out;
                    for (int k = 0; k < n->n_out; ++k) w->grad[out][k] = sd[k];
                } else {
                    double l = loss_one(n, w->val[out], ycls, yreg, b, dz);
                    lt[tid] += l * scale;
                    /* exact mode: the seed carries the 1/(S·B) scale; emulation: the unscaled
                     * seed is what the bf16 operand rounds, the scale is applied at accumulation */
                    for (int k = 0; k < n->n_out; ++k) w->grad[out][k] = emu_act ? dz[k] : dz[k] * scale;
                }
                backward_one(n, W, w, dWt + (size_t)tid * P, emu_act ? scale : 1.0, emu_act,
                             tmps + (size_t)tid * maxbuf);
            }
        }
        /* fixed-order reduction over threads, then the sample accumulation */
        for (int t = 0; t < nthreads; ++t) {
            const double* d = dWt + (size_t)t * P;
            if (t == 0) continue;
            for (long i = 0; i < P; ++i) dWt[i] += d[i];
        }
        for (long i = 0; i < P; ++i) {
            acc[i] += dWt[i];
            acc[P + i] += dWt[i] * E[i];
        }
        for (int t = 0; t < nthreads; ++t) acc[2 * P] += lt[t];
    }
    for (int t = 0; t < nthreads; ++t) free(works[t].pool);
    free(works);
    free(tmps);
    free(sigma); free(W); free(E); free(dWt); free(lt);
    return 0;
}

int orc_elbo_partial(const orc_model* m, const double* mu, const double* rho, const double* x,
                     const int* ycls, const double* yreg, int B_loc, int b_offset, int B_glob,
                     int S_glob, int s0, int s1, uint64_t seed, uint32_t step, int aug,
                     double* acc, int nthreads)
{
    return orc_elbo_partial_ex(m, mu, rho, x, ycls, yreg, B_loc, b_offset, B_glob, S_glob, s0, s1,
                               seed, step, aug, acc, nthreads, 0);
}

/*
 * Finalize (Alg. 1 l.10-12): from the summed partials produce loss, KL and gradients.
 *   grad_μ = acc_μ + μ/|D|;  grad_ρ = sigmoid(ρ)·(acc_ρ + (σ − 1/σ)/|D|)
 *   KL = ½ Σ (σ² + μ² − 1 − 2 ln σ);   loss = L_data + KL/|D|
 */
/* finalize of a P-parameter variational model (also the ViT oracle's, vit_oracle.c) */
int orc_finalize_p(long P, const double* mu, const double* rho, const double* acc, double D,
                   double* out_loss, double* out_kl, double* grad_mu, double* grad_rho)
{
    double kl = 0.0;
    for (long i = 0; i < P; ++i) {
        double sg = softplus(rho[i]);
        double ls = log_softplus(rho[i]);
        kl += 0.5 * (sg * sg + mu[i] * mu[i] - 1.0 - 2.0 * ls);
        grad_mu[i] = acc[i] + mu[i] / D;
        grad_rho[i] = sigmoid(rho[i]) * (acc[P + i] + (sg - 1.0 / sg) / D);
    }
    *out_kl = kl;
    *out_loss = acc[2 * P] + kl / D;
    return 0;
}

int orc_finalize(const orc_model* m, const double* mu, const double* rho, const double* acc,
                 double D, double* out_loss, double* out_kl, double* grad_mu, double* grad_rho)
{
    long P = orc_n_params(m);
    if (P < 0) return -1;
    if (m->mcd) {  /* MC dropout (R25): no variational distribution, no prior term */
        for (long i = 0; i < P; ++i) {
            grad_mu[i] = acc[i];
            grad_rho[i] = 0.0;
        }
        *out_kl = 0.0;
        *out_loss = acc[2 * P];
        return 0;
    }
    return orc_finalize_p(P, mu, rho, acc, D, out_loss, out_kl, grad_mu, grad_rho);
}

/*
 * Adam (Kingma & Ba 2015, Algorithm 1) — the optimizer Alg. 1 l.13 / Alg. 2 l.16 name
 * ("Update μ and σ using optimizer (e.g., Adam)"); SURVEY §8(f) f2.
 * Applied elementwise to θ ∈ {μ, ρ} (σ is parameterised by ρ, R1) with gradient g:
 *   m ← β1·m + (1 − β1)·g;   v ← β2·v + (1 − β2)·g²
 *   m̂ = m / (1 − β1^t);     v̂ = v / (1 − β2^t);     θ ← θ − α·m̂ / (√v̂ + ε)
 * t is the 1-based update count. fp64, in place.
 */
void orc_adam(long n, double* theta, const double* g, double* m, double* v, double alpha,
              double beta1, double beta2, double eps, int t)
{
    double bc1 = 1.0 - pow(beta1, (double)t);
    double bc2 = 1.0 - pow(beta2, (double)t);
    for (long i = 0; i < n; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
        double mhat = m[i] / bc1;
        double vhat = v[i] / bc2;
        theta[i] = theta[i] - alpha * mhat / (sqrt(vhat) + eps);
    }
}

/* Full single-process step: all S samples, all B examples. */
int orc_elbo_step(const orc_model* m, const double* mu, const double* rho, const double* x,
                  const int* ycls, const double* yreg, int B, int S, uint64_t seed,
                  uint32_t step, int aug, double D, double* out_loss, double* out_kl,
                  double* grad_mu, double* grad_rho, int nthreads)
{
    long P = orc_n_params(m);
    if (P < 0) return -1;
    double* acc = (double*)calloc((size_t)(2 * P + 1), sizeof(double));
    if (!acc) return -2;
    int rc = orc_elbo_partial(m, mu, rho, x, ycls, yreg, B, 0, B, S, 0, S, seed, step, aug, acc,
                              nthreads);
    if (!rc) rc = orc_finalize(m, mu, rho, acc, D, out_loss, out_kl, grad_mu, grad_rho);
    free(acc);
    return rc;
}

/*
 * Exact aggregation (§4.1 "an exact algorithm where the standard deviation
 * and mean are aggregated across multiple GPUs"): the data term is the loss
 * of the MEAN prediction over the S samples instead of the mean of per-sample losses:
 *   CE  ("cross-entropy loss on the (arithmetic) mean of the class probabilities"):
 *       p_s = softmax(z_s);  P̄_b = (1/S) Σ_s p_{s,b,y_b};  L_data = (1/B) Σ_b −ln P̄_b
 *   MSE ("MSE loss of the averaged predictions"):
 *       ȳ = (1/S) Σ_s z_s;  L_data = (1/(B·O)) Σ_{b,o} (ȳ_{b,o} − y_{b,o})²
 * loss = L_data + KL/|D|. Backward by the chain rule through the statistic:
 *   CE:  ∂L/∂z_{s,b,k} = (1/(S·B)) · (p_{s,b,y}/P̄_b) · (p_{s,b,k} − [k = y_b])
 *   MSE: ∂L/∂z_{s,b,o} = (2/(S·B·O)) · (ȳ_{b,o} − y_{b,o})
 * then the same per-sample backward and sample accumulation as orc_elbo_partial.
 */
static int forward_off(const orc_model* m, const double* mu, const double* rho, const double* x, int B,
                       int b_offset, int s0, int s1, uint64_t seed, uint32_t step, int aug, double* z_out,
                       int emu);

/* Shard statistic of the mean prediction for samples [s0,s1) and local examples [0,B_loc)
 * (global index b_offset + b): stats[b] = Σ_s p_{s,b,y_b} (CE, p_s = softmax(z_s)) or
 * stats[b·O + o] = Σ_s z_{s,b,o} (MSE). Summing the shards of all sample groups gives S·P̄_b or
 * S·ȳ_{b,o} (the statistic exchanged between forward and backward). */
int orc_mean_stats(const orc_model* m, const double* mu, const double* rho, const double* x,
                   const int* ycls, int B_loc, int b_offset, int s0, int s1, uint64_t seed,
                   uint32_t step, int aug, double* stats)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    const int O = net.n_out, S = s1 - s0;
    double* z = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * B_loc * O);
    if (!z) return -2;
    int rc = forward_off(m, mu, rho, x, B_loc, b_offset, s0, s1, seed, step, aug, z, 0);
    if (rc) return rc;
    const int w = m->loss == ORC_CE ? 1 : m->loss == ORC_GNLL ? 2 * O : O;
    for (long i = 0; i < (long)B_loc * w; ++i) stats[i] = 0.0;
    for (int s = 0; s < S; ++s)
        for (int b = 0; b < B_loc; ++b) {
            const double* zr = z + ((long)s * B_loc + b) * O;
            if (m->loss == ORC_CE) {
                double mx = zr[0];
                for (int k = 1; k < O; ++k) if (zr[k] > mx) mx = zr[k];
                double se = 0.0;
                for (int k = 0; k < O; ++k) se += exp(zr[k] - mx);
                stats[b] += exp(zr[ycls[b]] - mx) / se;
            } else if (m->loss == ORC_GNLL) {  /* Σ ŷ and Σ ŷ² (fp64) */
                for (int k = 0; k < O; ++k) {
                    stats[(long)b * 2 * O + k] += zr[k];
                    stats[(long)b * 2 * O + O + k] += zr[k] * zr[k];
                }
            } else {
                for (int k = 0; k < O; ++k) stats[(long)b * O + k] += zr[k];
            }
        }
    free(z);
    return 0;
}

/* Shard partial of the exact-aggregation step (the backward half): with the merged statistic
 * gstats (Σ over ALL S_glob samples, layout of orc_mean_stats) the per-sample gradient seeds
 *   CE:  ∂L/∂z_{s,b,k} = (1/(S·B)) · (p_{s,b,y}/P̄_b) · (p_{s,b,k} − [k = y_b]),  P̄_b = gstats[b]/S
 *   MSE: ∂L/∂z_{s,b,o} = (2/(S·B·O)) · (ȳ_{b,o} − y_{b,o}),                     ȳ = gstats/S
 * drive the per-sample backward of samples [s0,s1) into acc (as orc_elbo_partial); with
 * add_loss the shard's examples add their data loss, (1/B)Σ_b −ln P̄_b or (1/(B·O))Σ(ȳ − y)²,
 * to acc[2P] (one sample group adds it, so each example counts once). */
int orc_elbo_partial_mean(const orc_model* m, const double* mu, const double* rho, const double* x,
                          const int* ycls, const double* yreg, int B_loc, int b_offset, int B_glob,
                          int S_glob, int s0, int s1, uint64_t seed, uint32_t step, int aug,
                          const double* gstats, int add_loss, double* acc, int nthreads)
{
    long P = orc_n_params(m);
    if (P < 0) return -1;
    ONet net;
    if (build_net(m, &net)) return -1;
    const int O = net.n_out, S = s1 - s0;
    double* z = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * B_loc * O);
    double* seeds = (double*)calloc((size_t)S_glob * B_loc * O, sizeof(double)); /* indexed by global s */
    if (!z || !seeds) return -2;
    int rc = forward_off(m, mu, rho, x, B_loc, b_offset, s0, s1, seed, step, aug, z, 0);
    if (rc) return rc;
    double L = 0.0;
    for (int b = 0; b < B_loc; ++b) {
        if (m->loss == ORC_CE) {
            const int y = ycls[b];
            const double pbar = gstats[b] / S_glob;
            L += -log(pbar) / B_glob;
            for (int s = s0; s < s1; ++s) {
                const double* zr = z + ((long)(s - s0) * B_loc + b) * O;
                double mx = zr[0];
                for (int k = 1; k < O; ++k) if (zr[k] > mx) mx = zr[k];
                double se = 0.0;
                for (int k = 0; k < O; ++k) se += exp(zr[k] - mx);
                const double py = exp(zr[y] - mx) / se;
                double* sd = seeds + ((long)s * B_loc + b) * O;
                for (int k = 0; k < O; ++k)
                    sd[k] = (py / pbar) * (exp(zr[k] - mx) / se - (k == y ? 1.0 : 0.0)) /
                            ((double)S_glob * B_glob);
            }
        } else if (m->loss == ORC_GNLL) {
            /* Gaussian NLL of the predictive distribution (P:349 with P:148):
             *   m = (1/S)Σ ŷ_s,  v = (1/S)Σ (ŷ_s − m)² + ε_v,
             *   L = (1/(B·O)) Σ [ ½ ln(2π v) + (y − m)²/(2v) ]
             *   ∂L/∂ŷ_s = (1/(S·B·O)) [ (ŷ_s − m)/v − (y − m)/v − (y − m)²(ŷ_s − m)/v² ] */
            for (int k = 0; k < O; ++k) {
                const double mean = gstats[(long)b * 2 * O + k] / S_glob;
                const double v = gstats[(long)b * 2 * O + O + k] / S_glob - mean * mean + ORC_GNLL_EPS;
                const double d = yreg[(long)b * O + k] - mean;
                L += (0.5 * log(ORC_TWO_PI * v) + d * d / (2.0 * v)) / ((double)B_glob * O);
                for (int s = s0; s < s1; ++s) {
                    const double e = z[((long)(s - s0) * B_loc + b) * O + k] - mean;
                    seeds[((long)s * B_loc + b) * O + k] =
                        (e / v - d / v - d * d * e / (v * v)) / ((double)S_glob * B_glob * O);
                }
            }
        } else {
            for (int k = 0; k < O; ++k) {
                const double ybar = gstats[(long)b * O + k] / S_glob;
                const double d = ybar - yreg[(long)b * O + k];
                L += d * d / ((double)B_glob * O);
                for (int s = s0; s < s1; ++s)
                    seeds[((long)s * B_loc + b) * O + k] = 2.0 * d / ((double)S_glob * B_glob * O);
            }
        }
    }
    rc = elbo_partial_core(m, mu, rho, x, ycls, yreg, B_loc, b_offset, B_glob, S_glob, s0, s1, seed, step,
                           aug, acc, nthreads, 0, seeds);
    if (add_loss) acc[2 * P] += L;
    free(z);
    free(seeds);
    return rc;
}

/* The single-process exact step: the statistic of all S samples, then the backward. */
int orc_elbo_step_mean(const orc_model* m, const double* mu, const double* rho, const double* x,
                       const int* ycls, const double* yreg, int B, int S, uint64_t seed,
                       uint32_t step, int aug, double D, double* out_loss, double* out_kl,
                       double* grad_mu, double* grad_rho, int nthreads)
{
    long P = orc_n_params(m);
    if (P < 0) return -1;
    ONet net;
    if (build_net(m, &net)) return -1;
    const int w = m->loss == ORC_CE ? 1 : m->loss == ORC_GNLL ? 2 * net.n_out : net.n_out;
    double* st = (double*)malloc(sizeof(double) * (size_t)B * w);
    double* acc = (double*)calloc((size_t)(2 * P + 1), sizeof(double));
    if (!st || !acc) return -2;
    int rc = orc_mean_stats(m, mu, rho, x, ycls, B, 0, 0, S, seed, step, aug, st);
    if (!rc)
        rc = orc_elbo_partial_mean(m, mu, rho, x, ycls, yreg, B, 0, B, S, 0, S, seed, step, aug, st, 1, acc,
                                   nthreads);
    if (!rc) rc = orc_finalize(m, mu, rho, acc, D, out_loss, out_kl, grad_mu, grad_rho);
    free(st);
    free(acc);
    return rc;
}

/* Per-sample network outputs z[s][b][O] for samples [s0,s1) (no augmentation unless asked). */
int orc_forward_ex(const orc_model* m, const double* mu, const double* rho, const double* x, int B,
                   int s0, int s1, uint64_t seed, uint32_t step, int aug, double* z_out, int emu)
{
    return forward_off(m, mu, rho, x, B, 0, s0, s1, seed, step, aug, z_out, emu);
}

/* as orc_forward_ex for local examples whose global indices are b_offset + b (augmentation key) */
static int forward_off(const orc_model* m, const double* mu, const double* rho, const double* x, int B,
                       int b_offset, int s0, int s1, uint64_t seed, uint32_t step, int aug, double* z_out,
                       int emu)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    ONet* n = &net;
    long P = n->n_params;
    double* sigma = (double*)malloc(sizeof(double) * P);
    double* W = (double*)malloc(sizeof(double) * P);
    if (!sigma || !W) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    int nthreads = 1;
#ifdef _OPENMP
    nthreads = omp_get_max_threads();
#endif
    OWork* works = (OWork*)calloc((size_t)nthreads, sizeof(OWork));
    if (!works) return -2;
    for (int t = 0; t < nthreads; ++t)
        if (work_alloc(n, &works[t], 0)) return -2;
    for (int s = s0; s < s1; ++s) {
        sample_weights(n, mu, sigma, seed, step, (uint32_t)s, W, NULL, emu);
        #pragma omp parallel num_threads(nthreads)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            OWork* w = &works[tid];
            #pragma omp for schedule(static)
            for (int b = 0; b < B; ++b) {
                load_input(n, x, b, b_offset + b, seed, step, (uint32_t)s, aug, w->val[0]);
                drop_ctx(w, seed, step, (uint32_t)s, b_offset + b);
                int out = forward_one(n, W, w, emu);
                memcpy(z_out + ((long)(s - s0) * B + b) * n->n_out, w->val[out],
                       sizeof(double) * n->n_out);
            }
        }
    }
    for (int t = 0; t < nthreads; ++t) free(works[t].pool);
    free(works);
    free(sigma); free(W);
    return 0;
}

int orc_forward(const orc_model* m, const double* mu, const double* rho, const double* x, int B,
                int s0, int s1, uint64_t seed, uint32_t step, int aug, double* z_out)
{
    return orc_forward_ex(m, mu, rho, x, B, s0, s1, seed, step, aug, z_out, 0);
}

/*
 * Posterior predictive: per sample p_s = softmax(z_s) (CE) or z_s
 * (MSE); mean = (1/S) Σ p_s; var = (1/S) Σ (p_s − mean)² (population, reading R16). Two-pass.
 */
int orc_predict(const orc_model* m, const double* mu, const double* rho, const double* x, int B,
                int S, uint64_t seed, uint32_t step, double* mean, double* var)
{
    long O = (m->kind == ORC_MLP) ? m->widths[m->n_widths - 1] : m->n_classes;
    double* z = (double*)malloc(sizeof(double) * (size_t)S * B * O);
    if (!z) return -2;
    int rc = orc_forward(m, mu, rho, x, B, 0, S, seed, step, ORC_AUG_NONE, z);
    if (rc) { free(z); return rc; }
    if (m->loss == ORC_CE) {
        for (long r = 0; r < (long)S * B; ++r) {
            double* zr = z + r * O;
            double mx = zr[0];
            for (long k = 1; k < O; ++k) if (zr[k] > mx) mx = zr[k];
            double se = 0.0;
            for (long k = 0; k < O; ++k) se += exp(zr[k] - mx);
            for (long k = 0; k < O; ++k) zr[k] = exp(zr[k] - mx) / se;
        }
    }
    for (long i = 0; i < (long)B * O; ++i) {
        double acc = 0.0;
        for (int s = 0; s < S; ++s) acc += z[(long)s * B * O + i];
        double mu_i = acc / S;
        double v = 0.0;
        for (int s = 0; s < S; ++s) {
            double d = z[(long)s * B * O + i] - mu_i;
            v += d * d;
        }
        mean[i] = mu_i;
        var[i] = v / S;
    }
    free(z);
    return 0;
}

/* ======================================================================================
 * Part 3. Bulk helpers for the exhaustive EPS pins (tests/test_eps_oracle.py).
 * ====================================================================================== */

/* out[k-1] = LOG24(k·2^-24) for k = 1 .. 2^24 */
void orc_log24_all(float* out)
{
    #pragma omp parallel for schedule(static)
    for (long k = 1; k <= (1L << 24); ++k) out[k - 1] = orc_log24((float)k * 0x1p-24f);
}
/* c[v], s[v] = SINCOS2PI24(v) for v = 0 .. 2^24-1 */
void orc_sincos2pi24_all(float* c, float* s)
{
    #pragma omp parallel for schedule(static)
    for (long v = 0; v < (1L << 24); ++v) orc_sincos2pi24((uint32_t)v, &c[v], &s[v]);
}
/* Raw Philox outputs for n consecutive counters (x0 = c0 + i, others fixed). */
void orc_philox_fill(const uint32_t ctr[4], const uint32_t key[2], long n, uint32_t* out)
{
    #pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
        uint32_t c[4] = {ctr[0] + (uint32_t)i, ctr[1], ctr[2], ctr[3]};
        orc_philox4x32_10(c, key, out + 4 * i);
    }
}

/* Debug/test hook: the stored output of layer `layer` (after its activation and, with emu,
 * its bf16 rounding) for example b under sample s; returns the element count. */
long orc_layer_output(const orc_model* m, const double* mu, const double* rho, const double* x,
                      int b, int s, uint64_t seed, uint32_t step, int aug, int emu, int layer,
                      double* out)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    ONet* n = &net;
    long P = n->n_params;
    double* sigma = (double*)malloc(sizeof(double) * P);
    double* W = (double*)malloc(sizeof(double) * P);
    OWork w;
    if (!sigma || !W || work_alloc(n, &w, 0)) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    sample_weights(n, mu, sigma, seed, step, (uint32_t)s, W, NULL, emu);
    load_input(n, x, b, b, seed, step, (uint32_t)s, aug, w.val[0]);
    drop_ctx(&w, seed, step, (uint32_t)s, b);
    forward_one(n, W, &w, emu);
    long cnt = -3;
    for (int i = 0; i < n->n_ops; ++i)
        if (n->ops[i].type == OP_CONV && n->ops[i].layer == layer) {
            int d = n->ops[i].dst;
            cnt = buf_size(n, d);
            memcpy(out, w.val[d], sizeof(double) * (size_t)cnt);
        }
    free(w.pool); free(sigma); free(W);
    return cnt;
}

/* Debug/test hook: the (unscaled, masked) gradient dℓ/d(output of `layer`) for example b
 * under sample s after a full backward pass; emu as in orc_elbo_partial_ex. */
long orc_layer_grad(const orc_model* m, const double* mu, const double* rho, const double* x,
                    const int* ycls, const double* yreg, int b, int s, uint64_t seed, uint32_t step,
                    int aug, int emu, int layer, double* out)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    ONet* n = &net;
    long P = n->n_params;
    double* sigma = (double*)malloc(sizeof(double) * P);
    double* W = (double*)malloc(sizeof(double) * P);
    double* dW = (double*)calloc((size_t)P, sizeof(double));
    long maxbuf = 0;
    for (int q = 0; q < n->n_bufs; ++q) if (buf_size(n, q) > maxbuf) maxbuf = buf_size(n, q);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)maxbuf);
    OWork w;
    if (!sigma || !W || !dW || !tmp || work_alloc(n, &w, 1)) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    sample_weights(n, mu, sigma, seed, step, (uint32_t)s, W, NULL, emu);
    load_input(n, x, b, b, seed, step, (uint32_t)s, aug, w.val[0]);
    drop_ctx(&w, seed, step, (uint32_t)s, b);
    int outb = forward_one(n, W, &w, emu);
    double dz[4096];
    loss_one(n, w.val[outb], ycls, yreg, b, dz);
    for (int k = 0; k < n->n_out; ++k) w.grad[outb][k] = dz[k];
    backward_one(n, W, &w, dW, 1.0, emu, tmp);
    long cnt = -3;
    for (int i = 0; i < n->n_ops; ++i)
        if (n->ops[i].type == OP_CONV && n->ops[i].layer == layer) {
            int d = n->ops[i].dst;
            cnt = buf_size(n, d);
            memcpy(out, w.grad[d], sizeof(double) * (size_t)cnt);
        }
    free(w.pool); free(sigma); free(W); free(dW); free(tmp);
    return cnt;
}

/* Test hook: for example b under sample s, every layer's stored output (grad = 0) or the
 * unscaled dℓ/d(stored output) after a full backward pass (grad = 1), concatenated in layer
 * order — one forward (and backward) pass for all layers. Returns the element count. */
long orc_layer_dump(const orc_model* m, const double* mu, const double* rho, const double* x,
                    const int* ycls, const double* yreg, int b, int s, uint64_t seed, uint32_t step,
                    int aug, int emu, int grad, double* out)
{
    ONet net;
    if (build_net(m, &net)) return -1;
    ONet* n = &net;
    long P = n->n_params;
    double* sigma = (double*)malloc(sizeof(double) * P);
    double* W = (double*)malloc(sizeof(double) * P);
    double* dW = (double*)calloc((size_t)P, sizeof(double));
    long maxbuf = 0;
    for (int q = 0; q < n->n_bufs; ++q) if (buf_size(n, q) > maxbuf) maxbuf = buf_size(n, q);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)maxbuf);
    OWork w;
    if (!sigma || !W || !dW || !tmp || work_alloc(n, &w, 1)) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    sample_weights(n, mu, sigma, seed, step, (uint32_t)s, W, NULL, emu);
    load_input(n, x, b, b, seed, step, (uint32_t)s, aug, w.val[0]);
    drop_ctx(&w, seed, step, (uint32_t)s, b);
    int outb = forward_one(n, W, &w, emu);
    if (grad) {
        double dz[4096];
        loss_one(n, w.val[outb], ycls, yreg, b, dz);
        for (int k = 0; k < n->n_out; ++k) w.grad[outb][k] = dz[k];
        backward_one(n, W, &w, dW, 1.0, emu, tmp);
    }
    long cnt = 0;
    for (int l = 0; l < n->n_layers; ++l)
        for (int i = 0; i < n->n_ops; ++i)
            if (n->ops[i].type == OP_CONV && n->ops[i].layer == l) {
                int d = n->ops[i].dst;
                long sz = buf_size(n, d);
                memcpy(out + cnt, grad ? w.grad[d] : w.val[d], sizeof(double) * (size_t)sz);
                cnt += sz;
            }
    free(w.pool); free(sigma); free(W); free(dW); free(tmp);
    return cnt;
}
