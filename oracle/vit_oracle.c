/*
 * vit_oracle.c — the CPU oracle for the Bayesian ViT workload.
 *
 * TEST INFRASTRUCTURE ONLY (see bnn_oracle.c): plain fp64 loops, no blocking or fusion, no
 * code shared with the CUDA path. Built into the same liboracle.so as bnn_oracle.c, whose
 * EPS-v1 (orc_eps), augmentation (orc_aug_params) and finalize (orc_finalize_p) it calls.
 *
 * The model (use case 1; readings R27-R31):
 *   patches of P×P pixels (NHWC, element (dy, dx, c) at column (dy·P + dx)·C + c) →
 *   E = patch·W_pᵀ + b_p;  X_0 = [cls; E] + pos  (T = 1 + (H/P)(W/P) tokens of width D)
 *   for each of `depth` pre-norm encoder layers:
 *     H = LN(X; g1, b1);  [Q | K | V] = H·W_qkvᵀ + b_qkv  (head h: columns h·dh … h·dh+dh−1)
 *     A_h = softmax(Q_h K_hᵀ / √dh);  O_h = A_h V_h;  X ← X + O·W_projᵀ + b_proj
 *     H2 = LN(X; g2, b2);  U = H2·W_fc1ᵀ + b_fc1;  X ← X + GELU(U)·W_fc2ᵀ + b_fc2
 *   z = LN(X; g_f, b_f)[token 0]·W_headᵀ + b_head;  loss = CE(z, y)
 *   LN(x)_i = g_i (x_i − mean)/√(var + 1e-6) + b_i (biased variance over the D features);
 *   GELU(u) = ½u(1 + erf(u/√2)).
 * Every parameter tensor (weights, biases, LayerNorm g/b, cls, pos) is variational,
 * w_s = μ + softplus(ρ)·ε_s with ε_s = EPS-v1(seed, step, s, t, r, c) ("all weights";
 * readings R1, R3, R9). Tensor order t and shapes [rows, cols] (1-D tensors are [1, n]; pos is
 * [1, T·D], token-major):
 *   0 patch_w [D, P·P·C]   1 patch_b   2 cls [1, D]   3 pos [1, T·D]
 *   4 + 12l + {0 ln1_g, 1 ln1_b, 2 qkv_w [3D, D], 3 qkv_b, 4 proj_w [D, D], 5 proj_b,
 *              6 ln2_g, 7 ln2_b, 8 fc1_w [M, D], 9 fc1_b, 10 fc2_w [D, M], 11 fc2_b}
 *   4 + 12·depth + {0 lnf_g, 1 lnf_b, 2 head_w [O, D], 3 head_b}
 * Backward: the fp64 chain rule written out per operation below; the data-term gradient of
 * every parameter is accumulated per sample like bnn_oracle.c (acc_μ += Σ_s dW_s, acc_ρ +=
 * Σ_s ε_s ⊙ dW_s, both × 1/(S·B_glob)).
 *
 * Parity status: pinned by tests/test_vit_oracle.py — central finite differences of the
 * whole step (the network is smooth: no ReLU), an independent fp64 torch autograd
 * formulation (F.layer_norm, F.gelu, softmax), σ→0 = the deterministic ViT, and sample
 * averaging = brute force over single-sample runs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

float orc_eps(uint64_t seed, uint32_t step, uint32_t s, uint32_t t, uint32_t r, uint32_t c);
void orc_aug_params(uint64_t seed, uint32_t step, uint32_t s, uint32_t b, int* dx, int* dy, int* flip);

typedef struct {
    int in_h, in_w, in_c, patch;
    int dim, heads, depth, mlp, n_classes;
} orc_vit;

#define VIT_LN_EPS 1e-6

typedef struct {
    int T, D, M, Hd, dh, NP, PK, O;  /* tokens, width, mlp, heads, head dim, patches, patch K, classes */
    int nt;
    long off[4 + 12 * 64 + 4];
    int rows[4 + 12 * 64 + 4], cols[4 + 12 * 64 + 4];
    long P;
} VGeo;

static int vit_geo(const orc_vit* m, VGeo* g)
{
    if (m->patch <= 0 || m->in_h % m->patch || m->in_w % m->patch || m->heads <= 0 || m->dim % m->heads ||
        m->depth < 0 || m->depth > 64)
        return -1;
    g->NP = (m->in_h / m->patch) * (m->in_w / m->patch);
    g->T = 1 + g->NP;
    g->D = m->dim;
    g->M = m->mlp;
    g->Hd = m->heads;
    g->dh = m->dim / m->heads;
    g->PK = m->patch * m->patch * m->in_c;
    g->O = m->n_classes;
    int t = 0;
#define T_(r, c) do { g->rows[t] = (r); g->cols[t] = (c); ++t; } while (0)
    T_(g->D, g->PK); T_(1, g->D); T_(1, g->D); T_(1, g->T * g->D);
    for (int l = 0; l < m->depth; ++l) {
        T_(1, g->D); T_(1, g->D); T_(3 * g->D, g->D); T_(1, 3 * g->D); T_(g->D, g->D); T_(1, g->D);
        T_(1, g->D); T_(1, g->D); T_(g->M, g->D); T_(1, g->M); T_(g->D, g->M); T_(1, g->D);
    }
    T_(1, g->D); T_(1, g->D); T_(g->O, g->D); T_(1, g->O);
#undef T_
    g->nt = t;
    long off = 0;
    for (int i = 0; i < t; ++i) {
        g->off[i] = off;
        off += (long)g->rows[i] * g->cols[i];
    }
    g->P = off;
    return 0;
}

long orc_vit_n_params(const orc_vit* m)
{
    VGeo g;
    return vit_geo(m, &g) ? -1 : g.P;
}

int orc_vit_n_tensors(const orc_vit* m)
{
    VGeo g;
    return vit_geo(m, &g) ? -1 : g.nt;
}

/* info = {offset, rows, cols} */
int orc_vit_tensor_info(const orc_vit* m, int t, long* info)
{
    VGeo g;
    if (vit_geo(m, &g) || t < 0 || t >= g.nt) return -1;
    info[0] = g.off[t];
    info[1] = g.rows[t];
    info[2] = g.cols[t];
    return 0;
}

static double softplus(double r) { return (r > 0 ? r : 0.0) + log1p(exp(-fabs(r))); }

/* w_s = μ + σ ε_s for every parameter of global sample s (ε fp32 bits widened). eps_out keeps ε. */
/* BF16 mode's sampled weight (reading R14): RN_bf16(fma_f32(σ, ε, μ)) — used only by
 * the conditioning probe (emu_w = 1), the exact oracle keeps fp64 weights */
static double bf16_weight(double mu, double sigma, double e)
{
    float w = fmaf((float)sigma, (float)e, (float)mu);
    uint32_t u;
    memcpy(&u, &w, 4);
    uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
    memcpy(&w, &u, 4);
    return (double)w;
}

static int g_emu_w = 0;

static void vit_sample(const VGeo* g, const double* mu, const double* sigma, uint64_t seed, uint32_t step,
                       uint32_t s, double* W, double* eps_out)
{
    for (int t = 0; t < g->nt; ++t) {
        #pragma omp parallel for schedule(static)
        for (long r = 0; r < g->rows[t]; ++r)
            for (long c = 0; c < g->cols[t]; ++c) {
                long i = g->off[t] + r * g->cols[t] + c;
                double e = (double)orc_eps(seed, step, s, (uint32_t)t, (uint32_t)r, (uint32_t)c);
                eps_out[i] = e;
                W[i] = g_emu_w ? bf16_weight(mu[i], sigma[i], e) : mu[i] + sigma[i] * e;
            }
    }
}

/* ---------------------------------------------------------------- forward building blocks */
/* y[t][o] = Σ_k x[t][k] W[o][k] + b[o]   (W row-major [O][K]) */
static void linear(const double* x, int T, int K, const double* W, const double* b, int O, double* y)
{
    for (int t = 0; t < T; ++t)
        for (int o = 0; o < O; ++o) {
            double a = b[o];
            for (int k = 0; k < K; ++k) a += x[(long)t * K + k] * W[(long)o * K + k];
            y[(long)t * O + o] = a;
        }
}

/* LayerNorm over D features per token; xhat and rstd kept for the backward */
static void layernorm(const double* x, int T, int D, const double* gam, const double* bet, double* y,
                      double* xhat, double* rstd)
{
    for (int t = 0; t < T; ++t) {
        const double* xr = x + (long)t * D;
        double mean = 0.0;
        for (int i = 0; i < D; ++i) mean += xr[i];
        mean /= D;
        double var = 0.0;
        for (int i = 0; i < D; ++i) var += (xr[i] - mean) * (xr[i] - mean);
        var /= D;
        double rs = 1.0 / sqrt(var + VIT_LN_EPS);
        rstd[t] = rs;
        for (int i = 0; i < D; ++i) {
            double xh = (xr[i] - mean) * rs;
            xhat[(long)t * D + i] = xh;
            y[(long)t * D + i] = gam[i] * xh + bet[i];
        }
    }
}

static double gelu(double u) { return 0.5 * u * (1.0 + erf(u / sqrt(2.0))); }
static double gelu_d(double u)
{
    const double inv_sqrt2pi = 0.39894228040143267794;
    return 0.5 * (1.0 + erf(u / sqrt(2.0))) + u * inv_sqrt2pi * exp(-0.5 * u * u);
}

/* per-(sample, example) activations kept for the backward */
typedef struct {
    double *P, *X0;                                   /* patches [NP][PK], embedded tokens [T][D] */
    double **Xin, **H1, **xh1, **rs1, **QKV, **Att, **Ob, **Xmid, **H2, **xh2, **rs2, **U, **A;
    double *Xout, *Hf, *xhf, *rsf, *z;
} VAct;

static int act_alloc(const VGeo* g, int depth, VAct* a)
{
    int T = g->T, D = g->D, M = g->M;
    memset(a, 0, sizeof(*a));
    a->P = malloc(sizeof(double) * (size_t)g->NP * g->PK);
    a->X0 = malloc(sizeof(double) * (size_t)T * D);
    double*** fields[] = {&a->Xin, &a->H1, &a->xh1, &a->rs1, &a->QKV, &a->Att, &a->Ob,
                          &a->Xmid, &a->H2, &a->xh2, &a->rs2, &a->U, &a->A};
    size_t sz[] = {(size_t)T * D, (size_t)T * D, (size_t)T * D, (size_t)T, (size_t)T * 3 * D,
                   (size_t)g->Hd * T * T, (size_t)T * D, (size_t)T * D, (size_t)T * D, (size_t)T * D,
                   (size_t)T, (size_t)T * M, (size_t)T * M};
    for (int f = 0; f < 13; ++f) {
        *fields[f] = calloc((size_t)(depth > 0 ? depth : 1), sizeof(double*));
        if (!*fields[f]) return -1;
        for (int l = 0; l < depth; ++l) {
            (*fields[f])[l] = malloc(sizeof(double) * sz[f]);
            if (!(*fields[f])[l]) return -1;
        }
    }
    a->Xout = malloc(sizeof(double) * (size_t)T * D);
    a->Hf = malloc(sizeof(double) * (size_t)T * D);
    a->xhf = malloc(sizeof(double) * (size_t)T * D);
    a->rsf = malloc(sizeof(double) * (size_t)T);
    a->z = malloc(sizeof(double) * (size_t)g->O);
    return (a->P && a->X0 && a->Xout && a->Hf && a->xhf && a->rsf && a->z) ? 0 : -1;
}

static void act_free(int depth, VAct* a)
{
    double** fields[] = {a->Xin, a->H1, a->xh1, a->rs1, a->QKV, a->Att, a->Ob,
                         a->Xmid, a->H2, a->xh2, a->rs2, a->U, a->A};
    for (int f = 0; f < 13; ++f) {
        if (!fields[f]) continue;
        for (int l = 0; l < depth; ++l) free(fields[f][l]);
        free(fields[f]);
    }
    free(a->P); free(a->X0); free(a->Xout); free(a->Hf); free(a->xhf); free(a->rsf); free(a->z);
}

/* the (augmented) image of local example b → patches [NP][PK] */
static void patchify(const orc_vit* m, const VGeo* g, const double* x, int b_local, int b_global,
                     uint64_t seed, uint32_t step, uint32_t s, int aug, double* P)
{
    int H = m->in_h, W = m->in_w, C = m->in_c, p = m->patch;
    const double* src = x + (long)b_local * H * W * C;
    int dx = 4, dy = 4, flip = 0;
    if (aug) orc_aug_params(seed, step, s, (uint32_t)b_global, &dx, &dy, &flip);
    int pw = W / p;
    for (int py = 0; py < H / p; ++py)
        for (int px = 0; px < pw; ++px)
            for (int ddy = 0; ddy < p; ++ddy)
                for (int ddx = 0; ddx < p; ++ddx)
                    for (int c = 0; c < C; ++c) {
                        int i = py * p + ddy, j = px * p + ddx;  /* pixel of the augmented image */
                        int jj = flip ? W - 1 - j : j;
                        int si = i + dy - 4, sj = jj + dx - 4;
                        double v = (si >= 0 && si < H && sj >= 0 && sj < W) ? src[((long)si * W + sj) * C + c] : 0.0;
                        P[(long)(py * pw + px) * g->PK + (ddy * p + ddx) * C + c] = v;
                    }
}

static void forward_one(const orc_vit* m, const VGeo* g, const double* W, VAct* a)
{
    int T = g->T, D = g->D, M = g->M, Hd = g->Hd, dh = g->dh;
    /* patch embedding, cls, pos */
    double* E = a->Xout;  /* scratch [NP][D] */
    linear(a->P, g->NP, g->PK, W + g->off[0], W + g->off[1], D, E);
    for (int i = 0; i < D; ++i) a->X0[i] = W[g->off[2] + i] + W[g->off[3] + i];
    for (int t = 1; t < T; ++t)
        for (int i = 0; i < D; ++i)
            a->X0[(long)t * D + i] = E[(long)(t - 1) * D + i] + W[g->off[3] + (long)t * D + i];
    const double* X = a->X0;
    for (int l = 0; l < m->depth; ++l) {
        const long* o = g->off + 4 + 12 * l;
        memcpy(a->Xin[l], X, sizeof(double) * (size_t)T * D);
        layernorm(X, T, D, W + o[0], W + o[1], a->H1[l], a->xh1[l], a->rs1[l]);
        linear(a->H1[l], T, D, W + o[2], W + o[3], 3 * D, a->QKV[l]);
        const double* Q = a->QKV[l];
        double sc = 1.0 / sqrt((double)dh);
        for (int h = 0; h < Hd; ++h) {
            double* Ah = a->Att[l] + (long)h * T * T;
            for (int i = 0; i < T; ++i) {
                double mx = -INFINITY;
                for (int j = 0; j < T; ++j) {
                    double sdot = 0.0;
                    for (int e = 0; e < dh; ++e)
                        sdot += Q[(long)i * 3 * D + h * dh + e] * Q[(long)j * 3 * D + D + h * dh + e];
                    Ah[(long)i * T + j] = sdot * sc;
                    if (Ah[(long)i * T + j] > mx) mx = Ah[(long)i * T + j];
                }
                double se = 0.0;
                for (int j = 0; j < T; ++j) {
                    Ah[(long)i * T + j] = exp(Ah[(long)i * T + j] - mx);
                    se += Ah[(long)i * T + j];
                }
                for (int j = 0; j < T; ++j) Ah[(long)i * T + j] /= se;
                for (int e = 0; e < dh; ++e) {
                    double acc = 0.0;
                    for (int j = 0; j < T; ++j) acc += Ah[(long)i * T + j] * Q[(long)j * 3 * D + 2 * D + h * dh + e];
                    a->Ob[l][(long)i * D + h * dh + e] = acc;
                }
            }
        }
        linear(a->Ob[l], T, D, W + o[4], W + o[5], D, a->Xmid[l]);
        for (long i = 0; i < (long)T * D; ++i) a->Xmid[l][i] += X[i];
        layernorm(a->Xmid[l], T, D, W + o[6], W + o[7], a->H2[l], a->xh2[l], a->rs2[l]);
        linear(a->H2[l], T, D, W + o[8], W + o[9], M, a->U[l]);
        for (long i = 0; i < (long)T * M; ++i) a->A[l][i] = gelu(a->U[l][i]);
        linear(a->A[l], T, M, W + o[10], W + o[11], D, a->Xout);  /* X ← X_mid + MLP(LN2(X_mid)) */
        for (long i = 0; i < (long)T * D; ++i) a->Xout[i] += a->Xmid[l][i];
        X = a->Xout;
    }
    if (m->depth == 0) memcpy(a->Xout, a->X0, sizeof(double) * (size_t)T * D);
    const long* f = g->off + 4 + 12 * m->depth;
    layernorm(a->Xout, T, D, W + f[0], W + f[1], a->Hf, a->xhf, a->rsf);
    linear(a->Hf, 1, D, W + f[2], W + f[3], g->O, a->z);
}

/* ---------------------------------------------------------------- backward building blocks */
/* y = x·Wᵀ + b: dx = dy·W (accumulated into dx if given), dW += dyᵀ x, db += Σ_t dy */
static void linear_bwd(const double* x, int T, int K, const double* W, int O, const double* dy, double* dx,
                       double* dW, double* db)
{
    if (dx)
        for (int t = 0; t < T; ++t)
            for (int k = 0; k < K; ++k) {
                double a = 0.0;
                for (int o = 0; o < O; ++o) a += dy[(long)t * O + o] * W[(long)o * K + k];
                dx[(long)t * K + k] += a;
            }
    for (int o = 0; o < O; ++o) {
        for (int k = 0; k < K; ++k) {
            double a = 0.0;
            for (int t = 0; t < T; ++t) a += dy[(long)t * O + o] * x[(long)t * K + k];
            dW[(long)o * K + k] += a;
        }
        double a = 0.0;
        for (int t = 0; t < T; ++t) a += dy[(long)t * O + o];
        db[o] += a;
    }
}

/* y = g ⊙ x̂ + b, x̂ = (x − mean)·rstd: dx += rstd·(dx̂ − mean(dx̂) − x̂·mean(dx̂ ⊙ x̂)), dx̂ = dy ⊙ g */
static void layernorm_bwd(int T, int D, const double* gam, const double* xhat, const double* rstd,
                          const double* dy, double* dx, double* dg, double* db)
{
    for (int t = 0; t < T; ++t) {
        const double* dyr = dy + (long)t * D;
        const double* xh = xhat + (long)t * D;
        double m1 = 0.0, m2 = 0.0;
        for (int i = 0; i < D; ++i) {
            double dxh = dyr[i] * gam[i];
            m1 += dxh;
            m2 += dxh * xh[i];
            dg[i] += dyr[i] * xh[i];
            db[i] += dyr[i];
        }
        m1 /= D;
        m2 /= D;
        for (int i = 0; i < D; ++i) dx[(long)t * D + i] += rstd[t] * (dyr[i] * gam[i] - m1 - xh[i] * m2);
    }
}

/* dW: the per-sample parameter gradient (layout of the parameter vector); dz: dℓ/dz (unscaled) */
static void backward_one(const orc_vit* m, const VGeo* g, const double* W, VAct* a, const double* dz, double* dW,
                         double* tmp)
{
    int T = g->T, D = g->D, M = g->M, Hd = g->Hd, dh = g->dh;
    double* dX = tmp;                           /* [T][D] gradient of the residual stream */
    double* dH = dX + (long)T * D;              /* [T][D] */
    double* dQKV = dH + (long)T * D;            /* [T][3D] */
    double* dO = dQKV + (long)T * 3 * D;        /* [T][D] */
    double* dU = dO + (long)T * D;              /* [T][M] */
    double* dP = dU + (long)T * M;              /* [T] scratch */
    const long* f = g->off + 4 + 12 * m->depth;
    /* head on token 0, final LN */
    memset(dH, 0, sizeof(double) * (size_t)T * D);
    linear_bwd(a->Hf, 1, D, W + f[2], g->O, dz, dH, dW + f[2], dW + f[3]);
    memset(dX, 0, sizeof(double) * (size_t)T * D);
    layernorm_bwd(1, D, W + f[0], a->xhf, a->rsf, dH, dX, dW + f[0], dW + f[1]);
    for (int l = m->depth - 1; l >= 0; --l) {
        const long* o = g->off + 4 + 12 * l;
        /* X_out = X_mid + GELU(U)·W_fc2ᵀ + b_fc2 */
        double* dA = dU;
        memset(dA, 0, sizeof(double) * (size_t)T * M);
        linear_bwd(a->A[l], T, M, W + o[10], D, dX, dA, dW + o[10], dW + o[11]);
        for (long i = 0; i < (long)T * M; ++i) dU[i] = dA[i] * gelu_d(a->U[l][i]);
        memset(dH, 0, sizeof(double) * (size_t)T * D);
        linear_bwd(a->H2[l], T, D, W + o[8], M, dU, dH, dW + o[8], dW + o[9]);
        layernorm_bwd(T, D, W + o[6], a->xh2[l], a->rs2[l], dH, dX, dW + o[6], dW + o[7]);  /* dX = dX_mid */
        /* X_mid = X_in + O·W_projᵀ + b_proj */
        memset(dO, 0, sizeof(double) * (size_t)T * D);
        linear_bwd(a->Ob[l], T, D, W + o[4], D, dX, dO, dW + o[4], dW + o[5]);
        /* attention, per head: O_h = A_h V_h, A_h = softmax(S_h), S_h = Q_h K_hᵀ / √dh */
        memset(dQKV, 0, sizeof(double) * (size_t)T * 3 * D);
        const double* QKV = a->QKV[l];
        double sc = 1.0 / sqrt((double)dh);
        for (int h = 0; h < Hd; ++h) {
            const double* Ah = a->Att[l] + (long)h * T * T;
            for (int i = 0; i < T; ++i) {
                /* dA_ij = dO_i · V_j ; dS_ij = A_ij (dA_ij − Σ_k A_ik dA_ik) */
                double rowdot = 0.0;
                for (int j = 0; j < T; ++j) {
                    double d = 0.0;
                    for (int e = 0; e < dh; ++e) d += dO[(long)i * D + h * dh + e] * QKV[(long)j * 3 * D + 2 * D + h * dh + e];
                    dP[j] = d;
                    rowdot += Ah[(long)i * T + j] * d;
                }
                for (int j = 0; j < T; ++j) {
                    double dS = Ah[(long)i * T + j] * (dP[j] - rowdot) * sc;
                    double aij = Ah[(long)i * T + j];
                    for (int e = 0; e < dh; ++e) {
                        /* dV_j += A_ij dO_i ; dQ_i += dS_ij K_j ; dK_j += dS_ij Q_i */
                        dQKV[(long)j * 3 * D + 2 * D + h * dh + e] += aij * dO[(long)i * D + h * dh + e];
                        dQKV[(long)i * 3 * D + h * dh + e] += dS * QKV[(long)j * 3 * D + D + h * dh + e];
                        dQKV[(long)j * 3 * D + D + h * dh + e] += dS * QKV[(long)i * 3 * D + h * dh + e];
                    }
                }
            }
        }
        memset(dH, 0, sizeof(double) * (size_t)T * D);
        linear_bwd(a->H1[l], T, D, W + o[2], 3 * D, dQKV, dH, dW + o[2], dW + o[3]);
        layernorm_bwd(T, D, W + o[0], a->xh1[l], a->rs1[l], dH, dX, dW + o[0], dW + o[1]);  /* dX = dX_in */
    }
    /* X_0 = [cls; E] + pos, E = patch·W_pᵀ + b_p */
    for (int i = 0; i < D; ++i) dW[g->off[2] + i] += dX[i];
    for (long i = 0; i < (long)T * D; ++i) dW[g->off[3] + i] += dX[i];
    linear_bwd(a->P, g->NP, g->PK, W + g->off[0], D, dX + D, NULL, dW + g->off[0], dW + g->off[1]);
}

static double ce_loss(const double* z, int O, int y, double* dz)
{
    double mx = z[0];
    for (int k = 1; k < O; ++k) if (z[k] > mx) mx = z[k];
    double se = 0.0;
    for (int k = 0; k < O; ++k) se += exp(z[k] - mx);
    double lse = mx + log(se);
    for (int k = 0; k < O; ++k) dz[k] = exp(z[k] - lse) - (k == y ? 1.0 : 0.0);
    return lse - z[y];
}

/*
 * Partial data term over samples [s0, s1) and local examples [0, B_loc) (global b_offset + b):
 *   acc[0 .. P) += Σ_s Σ_b dℓ/dw / (S·B_glob); acc[P .. 2P) += Σ_s ε_s ⊙ Σ_b dℓ/dw / (S·B_glob);
 *   acc[2P] += Σ_s Σ_b ℓ / (S·B_glob). Fixed summation order for a fixed thread count.
 */
/* emu_w = 1: the sampled weights as the BF16 mode defines them (R14), everything else exact —
 * the conditioning probe of the BF16 tolerance (tests/test_conditioning.py) */
void orc_vit_set_emu_weights(int on) { g_emu_w = on; }

int orc_vit_elbo_partial(const orc_vit* m, const double* mu, const double* rho, const double* x, const int* ycls,
                         int B_loc, int b_offset, int B_glob, int S_glob, int s0, int s1, uint64_t seed,
                         uint32_t step, int aug, double* acc, int nthreads)
{
    VGeo g;
    if (vit_geo(m, &g)) return -1;
    long P = g.P;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    double* sigma = malloc(sizeof(double) * (size_t)P);
    double* W = malloc(sizeof(double) * (size_t)P);
    double* eps = malloc(sizeof(double) * (size_t)P);
    double* dWt = calloc((size_t)nthreads * P, sizeof(double));
    double* lt = calloc((size_t)nthreads, sizeof(double));
    if (!sigma || !W || !eps || !dWt || !lt) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    const double scale = 1.0 / ((double)S_glob * B_glob);
    long tmpn = (long)g.T * (g.D * 6 + g.M) + g.T;
    int rc = 0;
    for (int s = s0; s < s1; ++s) {
        vit_sample(&g, mu, sigma, seed, step, (uint32_t)s, W, eps);
        memset(dWt, 0, sizeof(double) * (size_t)nthreads * P);
        memset(lt, 0, sizeof(double) * (size_t)nthreads);
        #pragma omp parallel num_threads(nthreads)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            VAct a;
            double* tmp = malloc(sizeof(double) * (size_t)tmpn);
            double dz[64];
            if (act_alloc(&g, m->depth, &a) || !tmp || g.O > 64) {
                #pragma omp atomic write
                rc = -3;
            } else {
                #pragma omp for schedule(static)
                for (int b = 0; b < B_loc; ++b) {
                    patchify(m, &g, x, b, b_offset + b, seed, step, (uint32_t)s, aug, a.P);
                    forward_one(m, &g, W, &a);
                    lt[tid] += ce_loss(a.z, g.O, ycls[b], dz) * scale;
                    backward_one(m, &g, W, &a, dz, dWt + (size_t)tid * P, tmp);
                }
            }
            act_free(m->depth, &a);
            free(tmp);
        }
        if (rc) break;
        for (long i = 0; i < P; ++i) {
            double d = 0.0;
            for (int k = 0; k < nthreads; ++k) d += dWt[(size_t)k * P + i];
            acc[i] += d * scale;
            acc[P + i] += eps[i] * d * scale;
        }
        for (int k = 0; k < nthreads; ++k) acc[2 * P] += lt[k];
    }
    free(sigma); free(W); free(eps); free(dWt); free(lt);
    return rc;
}

/* logits [s1 − s0][B][O] of samples [s0, s1) (no augmentation) */
int orc_vit_forward(const orc_vit* m, const double* mu, const double* rho, const double* x, int B, int s0, int s1,
                    uint64_t seed, uint32_t step, int aug, double* out)
{
    VGeo g;
    if (vit_geo(m, &g)) return -1;
    long P = g.P;
    double* sigma = malloc(sizeof(double) * (size_t)P);
    double* W = malloc(sizeof(double) * (size_t)P);
    double* eps = malloc(sizeof(double) * (size_t)P);
    if (!sigma || !W || !eps) return -2;
    for (long i = 0; i < P; ++i) sigma[i] = softplus(rho[i]);
    int rc = 0;
    for (int s = s0; s < s1; ++s) {
        vit_sample(&g, mu, sigma, seed, step, (uint32_t)s, W, eps);
        #pragma omp parallel
        {
            VAct a;
            if (act_alloc(&g, m->depth, &a)) {
                #pragma omp atomic write
                rc = -3;
            } else {
                #pragma omp for schedule(static)
                for (int b = 0; b < B; ++b) {
                    patchify(m, &g, x, b, b, seed, step, (uint32_t)s, aug, a.P);
                    forward_one(m, &g, W, &a);
                    memcpy(out + ((long)(s - s0) * B + b) * g.O, a.z, sizeof(double) * (size_t)g.O);
                }
            }
            act_free(m->depth, &a);
        }
    }
    free(sigma); free(W); free(eps);
    return rc;
}
