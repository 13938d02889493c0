/*
 * include/nimble.h — C ABI of libnimble.so, the B200 (sm_100a) hot path of Nimble
 * (arXiv 2006.03031): shape functions, residue dispatch and dynamic-shape kernels.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * BJ:n = BASELINE.json line n.  The residue-dispatch rule is DISPATCH.md.
 *
 * Conventions (all entry points):
 *  - Every symbol is extern "C"; no C++ exception crosses the boundary.  Every
 *    entry point returns a nimble_status (0 = OK); on error the outputs are
 *    untouched, nothing is launched, and nimble_last_error() returns a
 *    thread-local message.
 *  - Ownership: the CALLER owns every buffer (inputs, outputs, workspace), sized
 *    from the shape functions BEFORE the call — the paper's shape_func -> alloc ->
 *    invoke_mut order (App. A; destination passing).  The
 *    library never allocates device memory on the hot path.
 *  - Device pointers are plain device addresses (cudaMalloc / torch storage).
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Kernels are asynchronous on `stream`; buffers must outlive the work.
 *    Asynchronous device faults surface at the caller's next synchronisation.
 *  - Layout: row-major with explicit leading dimensions `ld*` in ELEMENTS.
 *    bf16 paths use TMA: base pointers 16-byte aligned and ld*sizeof(elem) a
 *    multiple of 16, else NIMBLE_E_ALIGN.  fp32 paths require 16-byte aligned
 *    bases and ld % 4 == 0 (float4 loads), else NIMBLE_E_ALIGN.
 *  - The symbolic (Any) extent is M (dense), M/N/K (bmm, one symbol L),
 *    T (LSTM) or the level size (Tree-LSTM).  Extents must be >= 1 (SPEC S:170,
 *    S:438), else NIMBLE_E_EXTENT.  There is no CPU fallback: without a usable
 *    CUDA device the kernels return NIMBLE_E_CUDA.
 *  - Determinism: for a fixed dispatch the result is bitwise reproducible
 *    (split-K partials are reduced in rank order inside a thread-block cluster;
 *    no floating-point atomics).
 *  - Thread safety: all entry points are re-entrant; nimble_set_variant_limit is
 *    process-global and must be set before concurrent use.
 *  - Programmatic dependent launch (PDL, on unless NIMBLE_PDL=0): every kernel lets the
 *    next kernel on its stream start its prologue early, and the GEMMs (dense_dyn,
 *    dense_dyn_dev, dense_ln_dyn, dense_static) TMA-load the WEIGHT operand W of their
 *    first tiles BEFORE waiting for the preceding kernel (its bias, residual and x are
 *    read after the wait).  W must therefore not be written by the immediately preceding
 *    work on the same stream: weights are static per model (P:386-387 tiles the
 *    symbolic extent only).  Passing a just-computed activation as W needs NIMBLE_PDL=0
 *    or an event / other kernel in between.  bmm_dyn and attention wait before every load.
 */
#ifndef NIMBLE_H_
#define NIMBLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NIMBLE_ANY (-1) /* statically unknown extent, `Any` */

typedef enum {
    NIMBLE_OK = 0,
    NIMBLE_E_NULL = -1,        /* a required pointer is NULL */
    NIMBLE_E_RANK = -2,        /* wrong rank (reserved; ranks are fixed by the signatures) */
    NIMBLE_E_SHAPE = -3,       /* runtime type-relation violation: K or batch mismatch */
    NIMBLE_E_EXTENT = -4,      /* an extent < 1 or > 2^31-1 */
    NIMBLE_E_DTYPE = -5,       /* unknown dtype / epilogue code */
    NIMBLE_E_ALIGN = -6,       /* base or leading dimension misaligned for TMA / vector loads */
    NIMBLE_E_UNSUPPORTED = -7, /* a combination this build does not implement */
    NIMBLE_E_CUDA = -8         /* a CUDA runtime/driver call failed (message in nimble_last_error) */
} nimble_status;

typedef enum { NIMBLE_F32 = 0, NIMBLE_BF16 = 1 } nimble_dtype;

/* Fused epilogues (operator fusion of data-independent ops). */
typedef enum {
    NIMBLE_EPI_NONE = 0,          /* y = x W^T */
    NIMBLE_EPI_BIAS = 1,          /* y = x W^T + b */
    NIMBLE_EPI_BIAS_GELU = 2,     /* y = GELU_erf(x W^T + b)  (BERT FFN1) */
    NIMBLE_EPI_BIAS_RESIDUAL = 3  /* y = x W^T + b + residual (BERT O-proj, FFN2) */
} nimble_epilogue;

/* The dispatch record: exactly what the matching kernel entry point launches.
 * Field meanings are DISPATCH.md's.  family: 0 SIMT8 (fp32), 1 UMMA_T (bf16,
 * tokens on the UMMA-N slot), 2 UMMA_D (bf16 bmm with trans_b), 3 UMMA_T256 (bf16,
 * CTA pairs where they need fewer waves than family 1, DISPATCH.md), 4 UMMA_WS (bf16 dense, M <= 128: weight streaming, the K
 * splits of a feature tile one cluster).  variant -1 is the guarded fallback.
 * x = tile_t*k + r. */
typedef struct {
    int32_t family, tile_t, granule, n_classes, residue_class, variant, split_k;
    int32_t umma_m, umma_n_full, umma_n_tail;
    int64_t k, r;
    int32_t grid[3], cluster[3];
} nimble_dispatch;

/* ---------------------------------------------------------------------------
 * Shape functions — host, pure, data-independent mode.  They compute
 * the output shape for allocation and check the type relation at run time.
 * In/out are host int64 arrays.  A dim of NIMBLE_ANY switches to the compile-time
 * type relation: Any propagates, checks involving Any are deferred (gradual
 * typing); the bmm batch dim follows broadcast_rel.
 * dense:  x (M,K) x W (N,K)             -> (M,N)          K mismatch -> E_SHAPE
 * bmm:    A (B1,M,K) x B (B2,N,K)        -> (bcast(B1,B2),M,N)   trans_b = 0
 *         A (B1,M,K) x B (B2,K,N)        -> (bcast(B1,B2),M,N)   trans_b = 1
 * ------------------------------------------------------------------------- */
int nimble_shape_dense(const int64_t x_shape[2], const int64_t w_shape[2], int64_t out_shape[2]);
int nimble_shape_bmm(const int64_t a_shape[3], const int64_t b_shape[3], int trans_b,
                     int64_t out_shape[3]);

/* ---------------------------------------------------------------------------
 * Residue dispatch — host, pure (the generated dispatch function).  Returns
 * exactly the record the kernel entry point below will launch for these extents
 * under the current variant limit.  dt is a nimble_dtype.
 * ------------------------------------------------------------------------- */
int nimble_dispatch_dense(int64_t M, int64_t N, int64_t K, int dt, nimble_dispatch *out);
int nimble_dispatch_bmm(int64_t batch, int64_t M, int64_t N, int64_t K, int trans_b, int dt,
                        nimble_dispatch *out);

/* ---------------------------------------------------------------------------
 * Tuned schedules (Nimble §3.5 symbolic tuning: "tune with Any := 64, keep the
 * top-k, cross-evaluate on powers of two <= 256, pick the best average"; the procedure is
 * scripts/tune_symbolic.py).  A schedule registered for a bf16 dense op with weight
 * shape (N, K) replaces family 1's token tile t (the residue tile: x = t k + r, classes
 * ceil(r/16) in 0..t/16, so t/16 + 1 variants) and caps its split-K factor (t = 256 runs
 * without split-K: the fp32 exchange buffers would not fit shared memory); it applies to
 * nimble_dispatch_dense and nimble_dense_dyn with M < 2048 (at M >= 2048 the default rule,
 * family 1 or 3, runs; the static twin is not tuned).  tile_t in {32, 64, 128, 256} (0 removes the entry), split_max in {1, 2, 4, 8};
 * anything else -> NIMBLE_E_EXTENT.  Process-wide, thread-safe.  get: tile_t = 0 when no
 * schedule is registered (the default applies: t = 128, split cap 8 if K >= 2048, else 1).
 * ------------------------------------------------------------------------- */
int nimble_set_dense_schedule(int64_t N, int64_t K, int32_t tile_t, int32_t split_max);
int nimble_get_dense_schedule(int64_t N, int64_t K, int32_t *tile_t, int32_t *split_max);

/* c = total number of generated kernels ("dispatch/k"); 0 = all (default).
 * c < 0 -> E_EXTENT.  Process-global. */
int nimble_set_variant_limit(int c);
int nimble_get_variant_limit(void);
/* The dispatch record of the last successful kernel launch on the calling thread
 * ("instrumented variant-hit log"); E_NULL if none yet. */
int nimble_last_dispatch(nimble_dispatch *out);

/* ---------------------------------------------------------------------------
 * nimble_dense_dyn — y[M x N] = ep( x[M x K] . W[N x K]^T + bias ) (+ residual),
 * with M symbolic.  Device pointers; bias fp32 [N] (may be NULL only
 * for EPI_NONE); residual [M x ldr] of the output dtype (EPI_BIAS_RESIDUAL only).
 * dt = NIMBLE_F32: fp32 in/out, CUDA-core FFMA (SIMT8, t = 8 residue variants).
 * dt = NIMBLE_BF16: bf16 in/out, fp32 accumulation in TMEM (tcgen05 + TMA),
 *      output rounded to bf16 (RNE); rows >= M are never read (TMA bounds) nor
 *      written.  The dynamic extent is never padded.  With N % 8 != 0 the TMA stores of
 *      families 1 / 3 clip at 16-byte granularity: columns N .. ceil8(N)-1 of an output row
 *      (inside ldy, which the alignment rule makes >= ceil8(N)) may be overwritten.  With M <= 128 and no tuned
 *      schedule (family 4) the K splits' fp32 partials go through a library workspace
 *      owned by the calling STREAM (a pool of 16 per device, allocated on the stream's first
 *      family-4 launch, in relaxed capture mode inside a graph capture); more than 16
 *      streams share slots round-robin, and concurrent launches on two streams that share a
 *      slot are not supported.
 * ------------------------------------------------------------------------- */
int nimble_dense_dyn(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                     const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N,
                     int64_t K, int dt, int epi, void *stream);

/* nimble_dense_static — measurement baseline: the SAME kernel source as nimble_dense_dyn
 * instantiated with the extents as compile-time constants (the paper's static-shape
 * codegen, fig:sym-codegen P:696-703; "kernels compiled with a single static shape",
 * P:387).  Same arguments and dispatch record as nimble_dense_dyn.  Only compiled shapes
 * are available: fp32 with M in 1..64 (any N, K), bf16 with EPI_BIAS and (M, N, K) in the
 * table of umma_gemm.cu (BERT-large QKV/FFN2 shapes at M in {128, 384, 512, 513, 527,
 * 2048, 2049, 8192}, BERT-base shapes at M = 128); else NIMBLE_E_UNSUPPORTED. */
int nimble_dense_static(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                        const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N,
                        int64_t K, int dt, int epi, void *stream);

/* nimble_dense_ln_dyn — dense_dyn with the post-LN BERT sublayer tail fused in:
 *     y[i] = LayerNorm(x[i] W^T + bias + residual[i]) * gamma + beta,   i < M,
 * LayerNorm over the N features of each row (biased variance, eps inside the rsqrt;
 * DESIGN.md reading 10: post-LN, eps = 1e-12 in BERT).  Arguments as nimble_dense_dyn with
 * dt = NIMBLE_BF16 and the BIAS_RESIDUAL epilogue; gamma, beta: fp32 [N], 16-B aligned.
 * Where the residue dispatch picks the 2-CTA family (family 3), N = 1024 and K >= 2048
 * (a main loop long enough to hide the exchange) the LayerNorm runs in the GEMM epilogue: the 8 CTAs holding the four 256-feature quarters of a
 * 256-token tile exchange per-token (sum, sum of squares) partials through a library
 * workspace owned by the calling STREAM (a pool of 16 per device: launches on different
 * streams never share counters; two CUDA graphs captured on the same stream share one and
 * must not replay concurrently; more than 16 streams share slots round-robin).  The groups
 * spin on each other, so the group count is capped by the co-resident CTA pairs the
 * occupancy API reports (the two-launch form when none; also when the device's workspace
 * pool would first be allocated inside a graph capture).  The pre-LN sum is rounded to
 * bf16 first, as in the two-launch form.  Elsewhere: nimble_dense_dyn then nimble_layernorm in
 * place on y (same results up to the variance formula: fused = E[v^2] - mean^2 in fp32,
 * two-launch = two-pass).  Errors as nimble_dense_dyn; N % 8 != 0 or N > 4096 ->
 * E_UNSUPPORTED. */
int nimble_dense_ln_dyn(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                        const void *residual, int64_t ldr, const float *gamma, const float *beta, float eps,
                        void *y, int64_t ldy, int64_t M, int64_t N, int64_t K, void *stream);

/* nimble_dense_dyn_dev — device-resident extent and dispatch (the "upper bound" shape
 * function of P:269-271 plus on-device dispatch, so one captured CUDA graph serves every
 * extent; P:709-710 hides dispatch behind GPU execution).  bf16 only.  The caller
 * allocates by the bound M_max (1 <= M_max < 2048; nimble_shape_dense on (M_max, K) x
 * (N, K)); the true extent M is the int32 at M_dev (device memory, 1 <= M <= M_max, read
 * by the kernel after its grid-dependency wait, so an earlier kernel or copy on the stream
 * may write it).  The kernel runs the residue dispatch on the device.  With M_max <= 128 and
 * no schedule registered: family 4 of DISPATCH.md (weight streaming; its split S depends on
 * (N, K) only, so the bound's launch serves every M; the residue width and the record are
 * decided on the device; rows >= M of the token tile only feed unstored columns).  Otherwise
 * family 1 of DISPATCH.md with the token tile of the registered schedule (else 128) and the variant
 * limit c current at launch; split_k is the host rule's with the schedule's cap, else the
 * default cap evaluated at the bound M_max, when M_max fits one token tile (then it is the
 * same for every M <= M_max), else 1.  Writes y rows [0, M) only (the store's tensor
 * map is re-encoded on the device with extent M; rows [M, M_max) of y are untouched);
 * x rows in [M, M_max) are read but only feed unstored columns.  dispatch_dev: NULL or a
 * device nimble_dispatch that receives the device's dispatch decision.  A device extent
 * outside [1, M_max] traps (the error surfaces at the next synchronisation).  Uses a
 * library-owned ring of 64 per-launch tensor-map slot blocks per device: at most 64
 * nimble_dense_dyn_dev launches may be in flight at once. */
int nimble_dense_dyn_dev(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                         const void *residual, int64_t ldr, void *y, int64_t ldy, const int32_t *M_dev,
                         int64_t M_max, int64_t N, int64_t K, int epi, nimble_dispatch *dispatch_dev, void *stream);

/* ---------------------------------------------------------------------------
 * nimble_bmm_dyn — C[b] = alpha . A[b] . Bhat[b] over a strided batch (attention
 * heads), bf16 inputs, fp32 accumulation; out_dt = NIMBLE_F32 or NIMBLE_BF16.
 *   trans_b = 0: B[b] is [N x K] (row stride ldb), Bhat = B^T   (Q.K^T)
 *   trans_b = 1: B[b] is [K x N] (row stride ldb), Bhat = B     (P.V, MN-major B)
 * A[b] = A + b*strideA ([M x K], row stride lda); C[b] = C + b*strideC ([M x N],
 * row stride ldc); strides in elements, 16-byte multiples.  M, N, K may all be
 * the one symbol L; partial K tiles are zero-filled by TMA.  in_dt must
 * be NIMBLE_BF16 (E_UNSUPPORTED otherwise).
 * ------------------------------------------------------------------------- */
int nimble_bmm_dyn(const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                   int64_t strideB, int trans_b, void *C, int64_t ldc, int64_t strideC,
                   int64_t batch, int64_t M, int64_t N, int64_t K, float alpha, int in_dt,
                   int out_dt, void *stream);

/* nimble_bmm_static — measurement baseline for bmm_dyn: the same kernel source with
 * (M, N, K) compile-time constants (fig:sym-codegen P:696-703), for the attention-score form
 * only (trans_b = 0, fp32 output, alpha epilogue): (M, N, K) in {(128,128,64), (512,512,64),
 * (513,513,64), (2048,2048,64), (2049,2049,64)}; batch, strides and leading dims at run time.
 * Same arguments and dispatch record as nimble_bmm_dyn; other shapes / forms ->
 * NIMBLE_E_UNSUPPORTED. */
int nimble_bmm_static(const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                      int64_t strideB, int trans_b, void *C, int64_t ldc, int64_t strideC,
                      int64_t batch, int64_t M, int64_t N, int64_t K, float alpha, int in_dt,
                      int out_dt, void *stream);

/* ---------------------------------------------------------------------------
 * nimble_attention_varlen — fused attention over token-packed variable-length
 * requests: for request i = 0..R-1 (tokens
 * [seq_off[i], seq_off[i+1]) of the packed qkv), every head h:
 *     C_h = softmax( Q_h K_h^T * scale ) V_h,     L_i = seq_off[i+1] - seq_off[i]
 * qkv [T x ld_qkv] bf16 with row blocks Q | K | V of width heads*head_dim (BERT's
 * fused QKV projection output); out [T x ld_out] bf16, head h in columns
 * [h*head_dim, (h+1)*head_dim).  seq_off: DEVICE int32 [R+1], seq_off[0] = 0,
 * nondecreasing, seq_off[R] = T.  max_len >= every L_i.  One persistent launch (at
 * most 2 CTAs per SM walking a longest-request-first work list of (query tile, head,
 * request) items built on the device from seq_off); S and P stay on chip (TMEM /
 * smem; more than 1024 requests run as consecutive launches of 1024).  head_dim must be
 * 64 and max_len <= 8192 (E_UNSUPPORTED otherwise); qkv/out 16-byte aligned with
 * ld*2 % 16 == 0 (E_ALIGN).  seq_off is device data the host never reads: the kernel
 * validates it (seq_off[0] >= 0, nondecreasing, every L_i <= max_len, seq_off[R] <= T) and
 * traps (a sticky launch failure at the next synchronisation) instead of reading or
 * writing out of bounds.
 * ------------------------------------------------------------------------- */
int nimble_attention_varlen(const void *qkv, int64_t ld_qkv, int64_t T, const int32_t *seq_off, int32_t R,
                            int32_t max_len, int32_t heads, int32_t head_dim, float scale, void *out,
                            int64_t ld_out, void *stream);
/* nimble_attention_varlen_dev: the same op with the total token count on the device: T =
 * seq_off[R] is read by the kernel (T_max, the caller's allocation bound, sizes the launch
 * templates); each CTA re-encodes its Q/K and V tensor maps with extent T on the device, so
 * key rows at and beyond T read as zeros exactly as with a host T.  Request lengths, the
 * query-tile bound max_len and R keep their meaning.  Uses a library-owned ring of 64 slot
 * blocks per device: at most 64 such launches in flight. */
int nimble_attention_varlen_dev(const void *qkv, int64_t ld_qkv, int64_t T_max, const int32_t *seq_off, int32_t R,
                                int32_t max_len, int32_t heads, int32_t head_dim, float scale, void *out,
                                int64_t ld_out, void *stream);

/* ---------------------------------------------------------------------------
 * Row ops used around bmm_dyn in BERT (the paper is silent: DESIGN.md readings 8-10).
 * nimble_softmax_rows: P[b][i][j] = softmax_j(S[b][i][j]) over j < L, for i < rows;
 *   S fp32, P bf16; columns L..ldP-1 of P are written with 0 (so a following
 *   bmm may read up to a 64-aligned K without NaNs).  ldP >= L.
 * nimble_layernorm: Y = gamma (X - mean) / sqrt(var + eps) + beta over rows of
 *   length d, bf16 in/out, fp32 statistics, biased variance.
 * ------------------------------------------------------------------------- */
int nimble_softmax_rows(const float *S, int64_t ldS, int64_t strideS, void *P, int64_t ldP,
                        int64_t strideP, int64_t batch, int64_t rows, int64_t L, void *stream);
int nimble_layernorm(const void *X, int64_t ldx, const float *gamma, const float *beta, float eps,
                     void *Y, int64_t ldy, int64_t rows, int64_t d, void *stream);
/* nimble_layernorm_dev: nimble_layernorm over rows [0, *rows_dev) where the row count is
 * read on the device (device int32, 1 <= *rows_dev <= rows_max, else the kernel traps);
 * the launch covers rows_max (the upper bound the caller allocated).  Rows at and beyond
 * *rows_dev are untouched. */
int nimble_layernorm_dev(const void *X, int64_t ldx, const float *gamma, const float *beta, float eps, void *Y,
                         int64_t ldy, const int32_t *rows_dev, int64_t rows_max, int64_t d, void *stream);

/* ---------------------------------------------------------------------------
 * Fused dynamic-length LSTM layer (control flow as a device loop).
 * G [T x ldg] fp32 = X W_ih^T + (b_ih + b_hh), computed beforehand by
 * nimble_dense_dyn (the hoisted input GEMM).  W_hh [4H x ldw] fp32 in
 * PyTorch row blocks (i, f, g, o).  h0, c0 [H] (NULL -> zeros).  Writes
 * H_seq [T x ldh] (every h_t) and hT, cT [H].  One persistent cooperative kernel
 * runs all T steps with W_hh resident in shared memory and a grid barrier per
 * step.  workspace: device buffer of nimble_lstm_workspace_bytes(H) bytes.
 * ------------------------------------------------------------------------- */
size_t nimble_lstm_workspace_bytes(int64_t H);
int nimble_lstm_seq(const float *G, int64_t ldg, const float *W_hh, int64_t ldw, const float *h0,
                    const float *c0, float *H_seq, int64_t ldh, float *hT, float *cT, int64_t T,
                    int64_t H, void *workspace, void *stream);

/* Two stacked layers as ONE persistent wavefront kernel (layer 2 runs one step behind
 * layer 1; one grid barrier per step serves both, T + 1 barriers in all).  G1 [T x ldg] =
 * X W_ih1^T + (b_ih1 + b_hh1) (hoisted, nimble_dense_dyn); W_hh1, W_ih2, W_hh2 [4H x ldw]
 * (PyTorch row blocks i, f, g, o; layer 2's input is h1, so W_ih2 is [4H x H]); b2 [4H] =
 * b_ih2 + b_hh2; zero initial states.  Writes H1 [T x ldh], H2 [T x ldh] and hT, cT
 * [2 x H] (layer 0 then layer 1).  workspace: nimble_lstm2_workspace_bytes(H) bytes,
 * ZERO-FILLED by the caller before its first use; every call leaves it zero again (the last
 * CTA clears it), so no per-call memset sits on the hot path.  One workspace per concurrently
 * running call.  The weights are staged into shared memory before the kernel's
 * grid-dependency wait (PDL), overlapping the preceding input GEMM: W_hh1 / W_ih2 / W_hh2 must
 * not be written by the immediately preceding kernel on the stream.
 * H <= 1024 (E_UNSUPPORTED beyond: the weights must fit in shared memory). */
size_t nimble_lstm2_workspace_bytes(int64_t H);
/* The whole 2-layer forward in ONE launch: as nimble_lstm2_seq, with the layer-1 input
 * projection W_ih1 x_t + b1 computed inside the kernel ("the LSTM language model";
 * round-2 fusion of the hoisted input GEMM: each layer-1 CTA keeps its W_ih1 gate rows in shared
 * memory and computes x_t's projection while the previous step's h is being exchanged).
 * X [T x ldx] fp32 inputs (I features), W_ih1 [4H x ldwi], b1 [4H] = b_ih1 + b_hh1; the rest and
 * the workspace contract as nimble_lstm2_seq.  Register-resident weights only: H <= 672 and the
 * W_ih1 rows of a CTA in shared memory (I <= ~900 at H = 650), else NIMBLE_E_UNSUPPORTED (compose
 * nimble_dense_dyn + nimble_lstm2_seq).  W_ih1 / W_hh1 / W_ih2 / W_hh2 are read before the
 * kernel's grid-dependency wait: they must not be written by the immediately preceding kernel. */
int nimble_lstm2_forward(const float *X, int64_t ldx, int64_t I, const float *W_ih1, int64_t ldwi, const float *b1,
                         const float *W_hh1, const float *W_ih2, const float *W_hh2, int64_t ldw, const float *b2,
                         float *H1, float *H2, int64_t ldh, float *hT, float *cT, int64_t T, int64_t H,
                         void *workspace, void *stream);
int nimble_lstm2_seq(const float *G1, int64_t ldg, const float *W_hh1, const float *W_ih2, const float *W_hh2,
                     int64_t ldw, const float *b2, float *H1, float *H2, int64_t ldh, float *hT, float *cT,
                     int64_t T, int64_t H, void *workspace, void *stream);

/* ---------------------------------------------------------------------------
 * One Tree-LSTM level (binary N-ary cell; reading 13):
 * a level-batched dense_dyn over the M nodes of one height plus the cell epilogue.
 *   is_leaf = 1: A row of node m = A + a_rows[m]*lda (word vectors, K = I);
 *                W = W_l [3H x K] (gates i, o, u); c = s(i) tanh(u); h = s(o) tanh(c)
 *   is_leaf = 0: A row = A + a_rows[m]*lda holding [h_l | h_r] (K = 2H);
 *                W = U [5H x 2H] (gates i, f_l, f_r, o, u);
 *                c = s(i) tanh(u) + s(f_l) c_l + s(f_r) c_r,  [c_l | c_r] read from
 *                ccat + nodes[m]*ldcat;  h = s(o) tanh(c)
 * Writes h_out/c_out row nodes[m] (ld ldo) and, when parent_slot[m] = p*2+side >= 0,
 * h into hcat[p][side*H ...] and c into ccat[p][side*H ...] (ld ldcat): the
 * epilogue fills the parent's input row, so the next level needs no gather.
 * All fp32 device buffers; nodes, a_rows, parent_slot are device int32 [M].
 * ------------------------------------------------------------------------- */
int nimble_treelstm_level(const int32_t *nodes, const float *A, int64_t lda, const int32_t *a_rows,
                          const float *W, int64_t ldw, const float *bias, const int32_t *parent_slot,
                          float *hcat, float *ccat, int64_t ldcat, float *h_out, float *c_out,
                          int64_t ldo, int64_t M, int64_t K, int64_t H, int is_leaf, void *stream);

/* ---------------------------------------------------------------------------
 * A whole Tree-LSTM forest in ONE launch (same cell as nimble_treelstm_level; the level
 * loop of P:586's "small kernels plus control flow" runs on the device).  The schedule is
 * device data: nodes, rows, parent_slot are int32 [n_nodes] grouped by height, level l
 * occupying [level_off[l], level_off[l+1]) (level_off: device int32 [n_levels + 1]).
 * Level 0 holds exactly the leaves (height 0): A row = X + rows[m]*ldx (K = I), W = W_l
 * [3H x I] (row stride I).  Levels >= 1 hold internal nodes whose children sit in lower
 * levels: A row = hcat + rows[m]*ldcat (K = 2H), W = U [5H x 2H] (row stride 2H), [c_l|c_r]
 * from ccat + nodes[m]*ldcat.  Outputs and parent-slot writes as nimble_treelstm_level.
 * max_level = the largest level size (sizes the grid).  workspace: NIMBLE_TREE_WORKSPACE_BYTES
 * device bytes (level-barrier counter; reset by the call, stream-ordered).  All CTAs must be
 * co-resident (cooperative launch): a launch that cannot be returns NIMBLE_E_CUDA.
 * ------------------------------------------------------------------------- */
#define NIMBLE_TREE_WORKSPACE_BYTES 256
int nimble_treelstm_forest(const float *X, int64_t ldx, const float *W_l, const float *b_l, const float *U,
                           const float *b_u, int64_t I, int64_t H, const int32_t *level_off, int64_t n_levels,
                           int64_t max_level, const int32_t *nodes, const int32_t *rows, const int32_t *parent_slot,
                           float *hcat, float *ccat, int64_t ldcat, float *h_out, float *c_out, int64_t ldo,
                           void *workspace, void *stream);

/* ---------------------------------------------------------------------------
 * Request sharding (BJ:5): deterministic LPT partition of R requests of lengths
 * lens[R] over G ranks on cost(L) = 24 (25165824 L + 4096 L^2) (BERT-large flops):
 * sort by (cost desc, id asc), give each to the least-loaded rank (ties -> lowest).
 * Host arrays; owner[R] receives the rank of each request.
 * ------------------------------------------------------------------------- */
int64_t nimble_request_cost(int64_t L);
int nimble_partition_lpt(const int64_t *lens, int64_t R, int32_t G, int32_t *owner);

/* Instrumentation (not on the hot path): when buf != NULL, every later tcgen05 GEMM launch
 * writes 8 %globaltimer stamps (ns) per CTA into buf[cta*8 + slot] (device memory, caller-
 * sized): 0 start, 1 setup done, 2 first operands landed, 3 accumulator ready, 4 split-K
 * partial parked, 5 split-K slices received, 6 end.  NULL turns it off. */
int nimble_debug_trace(unsigned long long *buf);

/* Thread-local message for the last non-OK status ("" if none). */
const char *nimble_last_error(void);
/* Library version string. */
const char *nimble_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NIMBLE_H_ */
