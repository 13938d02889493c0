/*
 * oracle/oracle.c — the plain, slow, obviously-correct CPU oracle for the Nimble
 * (arXiv 2006.03031) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2006_03031_b200/) never links, imports or executes anything here, and this
 * file includes nothing from include/ or paper_2006_03031_b200/ (they share no code).
 *
 * Arithmetic: IEEE fp64, naive loops, ascending-k accumulation, no BLAS, compiled
 * without -ffast-math.  Inputs are the exact (bf16 / fp32) values the GPU sees,
 * widened to double by the caller.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * SURVEY §8(c) Oi = the oracle definition table; DESIGN.md "Readings" = where the
 * paper is silent.  Every function cites the passage it follows.
 *
 * Parity pins: see tests/test_oracle_*.py (closed forms, brute force, fp64 library
 * cross-checks, invariants).  Functions with no pin say "parity unpinned" — there
 * are none in this file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_ANY (-1)          /* statically unknown extent, `Any` */
#define ORC_OK 0
#define ORC_E_RANK (-2)
#define ORC_E_SHAPE (-3)
#define ORC_E_EXTENT (-4)
#define ORC_E_DTYPE (-5)
#define ORC_E_UNSUPPORTED (-7)

/* ------------------------------------------------------------------------- */
/* O1 — shape functions (P:230-238 broadcast_rel; "compute the output    */
/* shape ... and verify the type relation"; P:266-267 data independent).       */
/* ------------------------------------------------------------------------- */

/* broadcast_rel of one dimension pair.  The three `Any` rules are printed at
 * P:230-235; the static rules are numpy broadcasting (footnote at P:228).
 * (Any,d>1) -> d carries a runtime-check obligation (gradual typing). */
int orc_bcast(int64_t a, int64_t b, int64_t *out) {
    if (a == ORC_ANY && b == ORC_ANY) { *out = ORC_ANY; return ORC_OK; }   /* (Any,Any) -> Any */
    if (a == ORC_ANY) { *out = (b == 1) ? ORC_ANY : b; return ORC_OK; }    /* (Any,1)->Any, (Any,d)->d */
    if (b == ORC_ANY) { *out = (a == 1) ? ORC_ANY : a; return ORC_OK; }    /* symmetric */
    if (a < 1 || b < 1) return ORC_E_EXTENT;
    if (a == b) { *out = a; return ORC_OK; }
    if (a == 1) { *out = b; return ORC_OK; }
    if (b == 1) { *out = a; return ORC_OK; }
    return ORC_E_SHAPE;                                                    /* (d1,d2), d1!=d2, both >1 */
}

static int orc_dim_ok(int64_t d) { return d == ORC_ANY || d >= 1; }

/* dense: x (a0,a1) x W (w0,w1) -> (a0,w0); require a1 == w1 unless either is Any
 * (the check is deferred to run time).  W is [N x K] (reading 1). */
int orc_shape_dense(const int64_t x[2], const int64_t w[2], int64_t out[2]) {
    for (int i = 0; i < 2; i++)
        if (!orc_dim_ok(x[i]) || !orc_dim_ok(w[i])) return ORC_E_EXTENT;
    if (x[1] != ORC_ANY && w[1] != ORC_ANY && x[1] != w[1]) return ORC_E_SHAPE;
    out[0] = x[0];
    out[1] = w[0];
    return ORC_OK;
}

/* bmm: A (p0,p1,p2) x B (q0,q1,q2) -> (bcast(p0,q0), p1, trans_b ? q2 : q1);
 * K agreement p2 == (trans_b ? q1 : q2) unless Any (readings 2-3). */
int orc_shape_bmm(const int64_t a[3], const int64_t b[3], int trans_b, int64_t out[3]) {
    for (int i = 0; i < 3; i++)
        if (!orc_dim_ok(a[i]) || !orc_dim_ok(b[i])) return ORC_E_EXTENT;
    int64_t kb = trans_b ? b[1] : b[2];
    if (a[2] != ORC_ANY && kb != ORC_ANY && a[2] != kb) return ORC_E_SHAPE;
    int64_t bb;
    int st = orc_bcast(a[0], b[0], &bb);
    if (st != ORC_OK) return st;
    out[0] = bb;
    out[1] = a[1];
    out[2] = trans_b ? b[2] : b[1];
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O2 — the residue dispatch rule, written from DISPATCH.md.       */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t family, tile_t, granule, n_classes, residue_class, variant, split_k;
    int32_t umma_m, umma_n_full, umma_n_tail;
    int64_t k, r;
    int32_t grid[3], cluster[3];
} orc_dispatch;

static int orc_variant(int32_t cls, int32_t n_classes, int c) {
    /* c = total number of generated kernels (P:699 caption "generate k symbolic
     * kernels"); 0 = all.  Classes 0..c-2 specialised, the rest -> fallback (-1). */
    int cc = (c == 0 || c >= n_classes) ? n_classes : c;
    if (cc == n_classes) return cls;
    return (cls < cc - 1) ? cls : -1;
}

static int64_t orc_ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int32_t orc_split_cap(int64_t tiles, int64_t K, int32_t cap) {
    int64_t kb = orc_ceil_div(K, 64);
    int32_t s = 1;
    while (s < cap && tiles * 2 * s <= 148 && kb >= 8 * (int64_t)s) s *= 2;
    return s;
}

/* default split cap: split-K only for K >= 2048 (DISPATCH.md: below that the exchange of
 * fp32 partial tiles costs more than the shorter K loop saves, measured on B200; a cap that
 * depends on K alone keeps the split a function of the tile grid, so the dynamic-M result
 * stays bit-identical to pad-then-slice) */
static int32_t orc_default_cap(int64_t M, int64_t K) { (void)M; return K >= 2048 ? 8 : 1; }
static int32_t orc_split(int64_t tiles, int64_t M, int64_t K) { return orc_split_cap(tiles, K, orc_default_cap(M, K)); }

#define ORC_MAXEXT 2147483647LL

/* families 1 / 3, UMMA_T: tokens (symbolic M) on the UMMA-N slot, granule 16;
 * t = 128 (family 1, split-K allowed) or t = 256 (family 3, CTA pairs).  DISPATCH.md "Family 3":
 * family 3 exactly when its 256 x 256 tiles take fewer waves over 74 CTA pairs than family 1's
 * 128 x 128 tiles over 148 CTAs (round 2; measured rule, the paper leaves the tiling choice to
 * the schedule). */
static int orc_pairs_win(int64_t batch, int64_t M, int64_t N) {
    int64_t tiles_128 = orc_ceil_div(N, 128) * orc_ceil_div(M, 128) * batch;
    int64_t tiles_256 = orc_ceil_div(N, 256) * orc_ceil_div(M, 256) * batch;
    int64_t waves_1 = orc_ceil_div(tiles_128, 148), waves_3 = orc_ceil_div(tiles_256, 74);
    return waves_3 < waves_1;
}
/* tile_t / split_max: a tuned schedule for family 1 (DISPATCH.md "Tuned schedules",
 * P:392-406 three-step symbolic tuning picks them), used for M < 2048; tile_t = 0 -> the
 * default (128, cap 8 if K >= 2048, else 1). */
static int orc_umma_t_sched(int64_t batch, int64_t M, int64_t N, int64_t K, int c, int32_t tile_t,
                            int32_t split_max, orc_dispatch *d) {
    memset(d, 0, sizeof(*d));
    int tuned = (tile_t > 0 && M < 2048);
    int wide = !tuned && orc_pairs_win(batch, M, N);
    int32_t t = wide ? 256 : (tuned ? tile_t : 128);
    /* split-K exchanges two fp32 [128 x t] buffers through smem: only t <= 128 fits */
    int32_t cap = tuned ? (t <= 128 ? split_max : 1) : orc_default_cap(M, K);
    d->family = wide ? 3 : 1; d->tile_t = t; d->granule = 16; d->n_classes = t / 16 + 1;
    d->k = M / t; d->r = M % t;                      /* x = t k + r */
    d->residue_class = (int32_t)orc_ceil_div(d->r, 16);
    d->variant = orc_variant(d->residue_class, d->n_classes, c);
    d->umma_m = 128; d->umma_n_full = t;
    if (d->r == 0) d->umma_n_tail = 0;
    else d->umma_n_tail = (d->variant >= 0) ? 16 * d->residue_class : t;
    int64_t mt = orc_ceil_div(N, 128), nt = d->k + (d->r > 0);
    d->split_k = wide ? 1 : orc_split_cap(mt * nt * batch, K, cap);
    d->grid[0] = (int32_t)mt; d->grid[1] = (int32_t)nt; d->grid[2] = (int32_t)(batch * d->split_k);
    /* family 3 runs CTA pairs (tcgen05 cta_group::2): one 256-row MMA per pair */
    d->cluster[0] = wide ? 2 : 1; d->cluster[1] = 1; d->cluster[2] = d->split_k;
    if (wide) d->umma_m = 256;
    return ORC_OK;
}

static int orc_umma_t(int64_t batch, int64_t M, int64_t N, int64_t K, int c, orc_dispatch *d) {
    return orc_umma_t_sched(batch, M, N, K, c, 0, 8, d);
}

/* family 4, UMMA_WS (DISPATCH.md): a bf16 dense without a tuned schedule whose
 * (feature tile, token tile) units are few streams W over units x S CTAs,
 * S = min(ceil(K/64), floor(148 / units), 8) (at least 1) splits of K (the S splits of a unit
 * are one portable thread-block cluster, at most 8 CTAs); units = ceil(N/128) x ceil(M/128).
 * Taken when M <= 128 and ceil(N/128) <= 148, or when 128 < M <= 1024, K >= 2048 and S >= 2.
 * The residue split of M is family 1's (t = 128, granule 16, 9 classes). */
static int64_t orc_ws_splits(int64_t units, int64_t K) {
    int64_t kblocks = orc_ceil_div(K, 64);
    int64_t splits = 148 / units;
    if (splits > kblocks) splits = kblocks;
    if (splits > 8) splits = 8;                      /* one portable cluster per unit */
    if (splits < 1) splits = 1;
    return splits;
}

static int orc_ws_taken(int64_t M, int64_t N, int64_t K) {
    int64_t token_tiles = orc_ceil_div(M, 128), feature_tiles = orc_ceil_div(N, 128);
    if (token_tiles == 1) return feature_tiles <= 148;
    if (token_tiles > 8 || K < 2048) return 0;
    return orc_ws_splits(feature_tiles * token_tiles, K) >= 2;
}

static int orc_umma_ws(int64_t M, int64_t N, int64_t K, int c, orc_dispatch *d) {
    memset(d, 0, sizeof(*d));
    d->family = 4; d->tile_t = 128; d->granule = 16; d->n_classes = 9;
    d->k = M / 128; d->r = M % 128;                  /* x = t k + r */
    d->residue_class = (int32_t)orc_ceil_div(d->r, 16);
    d->variant = orc_variant(d->residue_class, 9, c);
    d->umma_m = 128; d->umma_n_full = 128;
    d->umma_n_tail = (d->r == 0) ? 0 : ((d->variant >= 0) ? 16 * d->residue_class : 128);
    int64_t feature_tiles = orc_ceil_div(N, 128), token_tiles = d->k + (d->r > 0);
    int64_t splits = orc_ws_splits(feature_tiles * token_tiles, K);
    d->split_k = (int32_t)splits;
    d->grid[0] = (int32_t)feature_tiles; d->grid[1] = (int32_t)token_tiles; d->grid[2] = (int32_t)splits;
    d->cluster[0] = 1; d->cluster[1] = 1; d->cluster[2] = 1;
    return ORC_OK;
}

int orc_dispatch_dense(int64_t M, int64_t N, int64_t K, int dt, int c, orc_dispatch *d) {
    if (M < 1 || N < 1 || K < 1 || M > ORC_MAXEXT || N > ORC_MAXEXT || K > ORC_MAXEXT) return ORC_E_EXTENT;
    if (c < 0) return ORC_E_EXTENT;
    memset(d, 0, sizeof(*d));
    if (dt == 0) {                       /* fp32 -> SIMT8, t = 8 */
        d->family = 0; d->tile_t = 8; d->granule = 1; d->n_classes = 8;
        d->k = M / 8; d->r = M % 8;      /* x = 8k + r */
        d->residue_class = (int32_t)d->r;
        d->variant = orc_variant(d->residue_class, 8, c);
        d->split_k = 1;
        d->grid[0] = (int32_t)orc_ceil_div(N, 32);    /* 32 output features per CTA */
        d->grid[1] = (int32_t)(d->k + (d->r > 0));
        d->grid[2] = 1;
        d->cluster[0] = d->cluster[1] = d->cluster[2] = 1;
        return ORC_OK;
    }
    if (dt != 1) return ORC_E_DTYPE;
    if (orc_ws_taken(M, N, K)) return orc_umma_ws(M, N, K, c, d);
    return orc_umma_t(1, M, N, K, c, d);
}

int orc_dispatch_dense_sched(int64_t M, int64_t N, int64_t K, int dt, int c, int32_t tile_t, int32_t split_max,
                             orc_dispatch *d) {
    if (tile_t == 0) return orc_dispatch_dense(M, N, K, dt, c, d);
    if (dt != 1) return ORC_E_DTYPE;                 /* schedules exist for the bf16 family only */
    if (!(tile_t == 32 || tile_t == 64 || tile_t == 128 || tile_t == 256)) return ORC_E_EXTENT;
    if (!(split_max == 1 || split_max == 2 || split_max == 4 || split_max == 8)) return ORC_E_EXTENT;
    if (M < 1 || N < 1 || K < 1 || M > ORC_MAXEXT || N > ORC_MAXEXT || K > ORC_MAXEXT) return ORC_E_EXTENT;
    if (c < 0) return ORC_E_EXTENT;
    return orc_umma_t_sched(1, M, N, K, c, tile_t, split_max, d);
}

int orc_dispatch_bmm(int64_t batch, int64_t M, int64_t N, int64_t K, int trans_b, int dt, int c,
                     orc_dispatch *d) {
    if (batch < 1 || batch > ORC_MAXEXT) return ORC_E_EXTENT;
    if (M < 1 || N < 1 || K < 1 || M > ORC_MAXEXT || N > ORC_MAXEXT || K > ORC_MAXEXT) return ORC_E_EXTENT;
    if (c < 0) return ORC_E_EXTENT;
    if (dt == 0) return ORC_E_UNSUPPORTED;
    if (dt != 1) return ORC_E_DTYPE;
    if (!trans_b) return orc_umma_t(batch, M, N, K, c, d);
    memset(d, 0, sizeof(*d));
    d->family = 2; d->tile_t = 128; d->granule = 128; d->n_classes = 2;
    d->k = M / 128; d->r = M % 128;
    d->residue_class = d->r > 0 ? 1 : 0;
    d->variant = orc_variant(d->residue_class, 2, c);
    d->umma_m = 128;
    int64_t nN = orc_ceil_div(N, 256);
    d->umma_n_full = (N >= 256) ? 256 : (int32_t)(16 * orc_ceil_div(N, 16));
    d->umma_n_tail = (int32_t)(16 * orc_ceil_div(N - 256 * (nN - 1), 16));
    int64_t mt = d->k + (d->r > 0);
    d->split_k = orc_split(mt * nN * batch, M, K);
    d->grid[0] = (int32_t)mt; d->grid[1] = (int32_t)nN; d->grid[2] = (int32_t)(batch * d->split_k);
    d->cluster[0] = 1; d->cluster[1] = 1; d->cluster[2] = d->split_k;
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O3 — dense: y*[m][n] = ep( sum_{k<K} x[m][k] W[n][k] + b[n] ) (+ res[m][n]). */
/* The residue variants compute exactly this function ("replace the  */
/* symbolic var x by 8k+r"); S:393 fixes the plain triple loop.  epi: 0 none,   */
/* 1 bias, 2 bias+GELU, 3 bias+residual (readings 8, 17).            */
/* Also returns D[m][n] = sum|x||W| + |b| + |res|, the error-bound denominator. */
/* ------------------------------------------------------------------------- */
double orc_gelu(double z) { return 0.5 * z * (1.0 + erf(z / sqrt(2.0))); }  /* exact erf GELU */

void orc_dense(const double *x, int64_t M, int64_t K, const double *W, int64_t N, const double *b,
               const double *res, int epi, double *y, double *D) {
    for (int64_t m = 0; m < M; m++) {
        for (int64_t n = 0; n < N; n++) {
            double acc = 0.0, den = 0.0;
            for (int64_t k = 0; k < K; k++) {          /* ascending k */
                acc += x[m * K + k] * W[n * K + k];
                den += fabs(x[m * K + k]) * fabs(W[n * K + k]);
            }
            if (epi >= 1 && b) { acc += b[n]; den += fabs(b[n]); }
            if (epi == 2) acc = orc_gelu(acc);
            if (epi == 3 && res) { acc += res[m * N + n]; den += fabs(res[m * N + n]); }
            y[m * N + n] = acc;
            if (D) D[m * N + n] = den;
        }
    }
}

/* O4 — bmm: C*[b][i][j] = alpha * sum_k A[bA][i][k] * Bhat[bB][j][k], Bhat = B
 * (trans_b = 0, B is [N x K]) or B^T (trans_b = 1, B is [K x N]); a batch of 1
 * broadcasts (readings 2-3).  One symbol L may stand for
 * M = N = K ("a single variable dimension for equivalent dynamic dims"). */
void orc_bmm(const double *A, int64_t bA, const double *B, int64_t bB, int64_t M, int64_t N, int64_t K,
             int trans_b, double alpha, double *C, double *D) {
    int64_t batch = bA > bB ? bA : bB;
    for (int64_t b = 0; b < batch; b++) {
        const double *a = A + (bA == 1 ? 0 : b) * M * K;
        const double *bb = B + (bB == 1 ? 0 : b) * N * K;
        for (int64_t i = 0; i < M; i++)
            for (int64_t j = 0; j < N; j++) {
                double acc = 0.0, den = 0.0;
                for (int64_t k = 0; k < K; k++) {
                    double bv = trans_b ? bb[k * N + j] : bb[j * K + k];
                    acc += a[i * K + k] * bv;
                    den += fabs(a[i * K + k]) * fabs(bv);
                }
                C[(b * M + i) * N + j] = alpha * acc;
                if (D) D[(b * M + i) * N + j] = fabs(alpha) * den;
            }
    }
}

/* ------------------------------------------------------------------------- */
/* O5 — row ops (BERT conventions; the paper is silent: DESIGN.md 8-10).       */
/* ------------------------------------------------------------------------- */
/* softmax_j(s) = exp(s_j - max s) / sum_j exp(s_j - max s), over rows of length L */
void orc_softmax_rows(const double *S, int64_t rows, int64_t L, double *P) {
    for (int64_t i = 0; i < rows; i++) {
        const double *s = S + i * L;
        double mx = s[0];
        for (int64_t j = 1; j < L; j++) if (s[j] > mx) mx = s[j];
        double sum = 0.0;
        for (int64_t j = 0; j < L; j++) sum += exp(s[j] - mx);
        for (int64_t j = 0; j < L; j++) P[i * L + j] = exp(s[j] - mx) / sum;
    }
}

/* LN(x) = gamma * (x - mu) / sqrt(var + eps) + beta, biased variance, eps 1e-12 */
void orc_layernorm(const double *X, int64_t rows, int64_t d, const double *gamma, const double *beta,
                   double eps, double *Y) {
    for (int64_t i = 0; i < rows; i++) {
        const double *x = X + i * d;
        double mu = 0.0;
        for (int64_t j = 0; j < d; j++) mu += x[j];
        mu /= (double)d;
        double var = 0.0;
        for (int64_t j = 0; j < d; j++) var += (x[j] - mu) * (x[j] - mu);
        var /= (double)d;
        double inv = 1.0 / sqrt(var + eps);
        for (int64_t j = 0; j < d; j++) Y[i * d + j] = gamma[j] * (x[j] - mu) * inv + beta[j];
    }
}

static double orc_sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

/* ------------------------------------------------------------------------- */
/* O6 — one LSTM layer over a runtime-length sequence (P:575-576;    */
/* gate order i,f,g,o and folded bias b = b_ih + b_hh: DESIGN.md reading 12).  */
/* for t: z = W_ih x_t + W_hh h_{t-1} + b; i,f,o = sigma, g = tanh;             */
/*        c_t = f*c_{t-1} + i*g;  h_t = o*tanh(c_t)                              */
/* h0/c0 may be NULL (zeros).  Hseq [T x H]; hT, cT [H].                        */
/* ------------------------------------------------------------------------- */
void orc_lstm_layer(const double *X, int64_t T, int64_t I, int64_t H, const double *W_ih,
                    const double *W_hh, const double *b, const double *h0, const double *c0,
                    double *Hseq, double *hT, double *cT) {
    double *h = (double *)malloc(sizeof(double) * H);
    double *c = (double *)malloc(sizeof(double) * H);
    double *z = (double *)malloc(sizeof(double) * 4 * H);
    for (int64_t j = 0; j < H; j++) { h[j] = h0 ? h0[j] : 0.0; c[j] = c0 ? c0[j] : 0.0; }
    for (int64_t t = 0; t < T; t++) {
        const double *x = X + t * I;
        for (int64_t r = 0; r < 4 * H; r++) {
            double acc = 0.0;
            for (int64_t k = 0; k < I; k++) acc += W_ih[r * I + k] * x[k];
            for (int64_t k = 0; k < H; k++) acc += W_hh[r * H + k] * h[k];
            z[r] = acc + b[r];
        }
        for (int64_t j = 0; j < H; j++) {
            double ig = orc_sigmoid(z[j]);
            double fg = orc_sigmoid(z[H + j]);
            double gg = tanh(z[2 * H + j]);
            double og = orc_sigmoid(z[3 * H + j]);
            c[j] = fg * c[j] + ig * gg;
            h[j] = og * tanh(c[j]);
            Hseq[t * H + j] = h[j];
        }
    }
    for (int64_t j = 0; j < H; j++) { if (hT) hT[j] = h[j]; if (cT) cT[j] = c[j]; }
    free(h); free(c); free(z);
}

/* ------------------------------------------------------------------------- */
/* O7 — binary N-ary Tree-LSTM (reading 13),       */
/* recursive post-order.  Node i is a leaf iff left[i] < 0; leaf word vector    */
/* X[word[i]] (dim I).  Leaf:  [i;o;u] = W_l x + b_l;  c = s(i) tanh(u);        */
/*                             h = s(o) tanh(c).                                 */
/* Internal: [i;fl;fr;o;u] = U [h_l; h_r] + b_u;                                 */
/*           c = s(i) tanh(u) + s(fl) c_l + s(fr) c_r;  h = s(o) tanh(c).         */
/* W_l [3H x I], U [5H x 2H].  Outputs Hn, Cn [n_nodes x H].                     */
/* ------------------------------------------------------------------------- */
typedef struct {
    const int32_t *left, *right, *word;
    const double *X, *W_l, *b_l, *U, *b_u;
    int64_t I, H;
    double *Hn, *Cn;
} orc_tree_ctx;

static void orc_tree_node(const orc_tree_ctx *t, int32_t i) {
    int64_t H = t->H;
    double *h = t->Hn + (int64_t)i * H, *c = t->Cn + (int64_t)i * H;
    if (t->left[i] < 0) {
        const double *x = t->X + (int64_t)t->word[i] * t->I;
        for (int64_t j = 0; j < H; j++) {
            double zi = t->b_l[j], zo = t->b_l[H + j], zu = t->b_l[2 * H + j];
            for (int64_t k = 0; k < t->I; k++) {
                zi += t->W_l[j * t->I + k] * x[k];
                zo += t->W_l[(H + j) * t->I + k] * x[k];
                zu += t->W_l[(2 * H + j) * t->I + k] * x[k];
            }
            c[j] = orc_sigmoid(zi) * tanh(zu);
            h[j] = orc_sigmoid(zo) * tanh(c[j]);
        }
        return;
    }
    int32_t l = t->left[i], r = t->right[i];
    orc_tree_node(t, l);                             /* post-order: children first */
    orc_tree_node(t, r);
    const double *hl = t->Hn + (int64_t)l * H, *hr = t->Hn + (int64_t)r * H;
    const double *cl = t->Cn + (int64_t)l * H, *cr = t->Cn + (int64_t)r * H;
    for (int64_t j = 0; j < H; j++) {
        double z[5];
        for (int g = 0; g < 5; g++) {
            const double *u = t->U + ((int64_t)g * H + j) * 2 * H;
            double acc = t->b_u[g * H + j];
            for (int64_t k = 0; k < H; k++) acc += u[k] * hl[k];
            for (int64_t k = 0; k < H; k++) acc += u[H + k] * hr[k];
            z[g] = acc;
        }
        c[j] = orc_sigmoid(z[0]) * tanh(z[4]) + orc_sigmoid(z[1]) * cl[j] + orc_sigmoid(z[2]) * cr[j];
        h[j] = orc_sigmoid(z[3]) * tanh(c[j]);
    }
}

void orc_treelstm(int32_t root, const int32_t *left, const int32_t *right, const int32_t *word,
                  const double *X, int64_t I, int64_t H, const double *W_l, const double *b_l,
                  const double *U, const double *b_u, double *Hn, double *Cn) {
    orc_tree_ctx t = {left, right, word, X, W_l, b_l, U, b_u, I, H, Hn, Cn};
    orc_tree_node(&t, root);
}

/* ------------------------------------------------------------------------- */
/* O8 — one post-LN BERT encoder layer ("BERT base";    */
/* DESIGN.md readings 8-10), composed of O3/O4/O5 with no intermediate rounding: */
/*  QKV = X Wqkv^T + bqkv;  S_h = Q_h K_h^T / sqrt(dh);  P_h = softmax(S_h);     */
/*  C_h = P_h V_h;  A = C Wo^T + bo + X;  H1 = LN1(A);                            */
/*  F = GELU(H1 W1^T + b1);  O = F W2^T + b2 + H1;  Y = LN2(O)                    */
/* ------------------------------------------------------------------------- */
void orc_bert_layer(const double *X, int64_t L, int64_t d, int64_t nh, int64_t f,
                    const double *Wqkv, const double *bqkv, const double *Wo, const double *bo,
                    const double *g1, const double *be1, const double *W1, const double *b1,
                    const double *W2, const double *b2, const double *g2, const double *be2,
                    double *Y) {
    int64_t dh = d / nh;
    double *QKV = (double *)malloc(sizeof(double) * L * 3 * d);
    double *Qh = (double *)malloc(sizeof(double) * L * dh);
    double *Kh = (double *)malloc(sizeof(double) * L * dh);
    double *Vh = (double *)malloc(sizeof(double) * L * dh);
    double *S = (double *)malloc(sizeof(double) * L * L);
    double *P = (double *)malloc(sizeof(double) * L * L);
    double *Ch = (double *)malloc(sizeof(double) * L * dh);
    double *C = (double *)malloc(sizeof(double) * L * d);
    double *A = (double *)malloc(sizeof(double) * L * d);
    double *H1 = (double *)malloc(sizeof(double) * L * d);
    double *F = (double *)malloc(sizeof(double) * L * f);
    double *O = (double *)malloc(sizeof(double) * L * d);
    orc_dense(X, L, d, Wqkv, 3 * d, bqkv, NULL, 1, QKV, NULL);
    for (int64_t h = 0; h < nh; h++) {
        for (int64_t i = 0; i < L; i++)
            for (int64_t e = 0; e < dh; e++) {
                Qh[i * dh + e] = QKV[i * 3 * d + h * dh + e];
                Kh[i * dh + e] = QKV[i * 3 * d + d + h * dh + e];
                Vh[i * dh + e] = QKV[i * 3 * d + 2 * d + h * dh + e];
            }
        orc_bmm(Qh, 1, Kh, 1, L, L, dh, 0, 1.0 / sqrt((double)dh), S, NULL);
        orc_softmax_rows(S, L, L, P);
        orc_bmm(P, 1, Vh, 1, L, dh, L, 1, 1.0, Ch, NULL);
        for (int64_t i = 0; i < L; i++)
            for (int64_t e = 0; e < dh; e++) C[i * d + h * dh + e] = Ch[i * dh + e];
    }
    orc_dense(C, L, d, Wo, d, bo, X, 3, A, NULL);
    orc_layernorm(A, L, d, g1, be1, 1e-12, H1);
    orc_dense(H1, L, d, W1, f, b1, NULL, 2, F, NULL);
    orc_dense(F, L, f, W2, d, b2, H1, 3, O, NULL);
    orc_layernorm(O, L, d, g2, be2, 1e-12, Y);
    free(QKV); free(Qh); free(Kh); free(Vh); free(S); free(P); free(Ch);
    free(C); free(A); free(H1); free(F); free(O);
}

/* ------------------------------------------------------------------------- */
/* O9 — deterministic LPT partition of a request stream over G ranks (BJ:5     */
/* "partitioned across the 8 GPUs ... each GPU running whole requests";         */
/* SURVEY §8(c) O9).  cost(L) = 24 (25165824 L + 4096 L^2) (BERT-large flops).   */
/* Sort by (cost desc, id asc); each request goes to the least-loaded rank,     */
/* ties to the lowest rank.  Plain O(R^2 + R G) selection — no heap.             */
/* ------------------------------------------------------------------------- */
int64_t orc_request_cost(int64_t L) { return 24 * (25165824LL * L + 4096LL * L * L); }

int orc_partition_lpt(const int64_t *lens, int64_t R, int32_t G, int32_t *owner) {
    if (G < 1 || R < 0) return ORC_E_EXTENT;
    for (int64_t i = 0; i < R; i++) if (lens[i] < 1) return ORC_E_EXTENT;
    char *done = (char *)calloc(R > 0 ? R : 1, 1);
    int64_t *load = (int64_t *)calloc(G, sizeof(int64_t));
    for (int64_t step = 0; step < R; step++) {
        int64_t best = -1;                             /* next request in (cost desc, id asc) */
        for (int64_t i = 0; i < R; i++) {
            if (done[i]) continue;
            if (best < 0 || orc_request_cost(lens[i]) > orc_request_cost(lens[best])) best = i;
        }
        int32_t g = 0;
        for (int32_t q = 1; q < G; q++) if (load[q] < load[g]) g = q;
        owner[best] = g;
        load[g] += orc_request_cost(lens[best]);
        done[best] = 1;
    }
    free(done); free(load);
    return ORC_OK;
}
