// Host-side launch descriptors shared between api.cu and the kernel translation units.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "nimble.h"

namespace nimble {

// Parameters of one tcgen05 GEMM launch (families UMMA_T / UMMA_D, DISPATCH.md).
//   D[i][j] = sum_k A[i][k] * B[j][k]   (i on the UMMA-M slot, j on the UMMA-N slot)
// transposed epilogue: out[b*stride + j*ld + i]  (lane = i = output feature; TMA store)
// direct epilogue:     out[b*stride + i*ld + j]  (row-major in i; vector stores)
struct UmmaParams {
    int32_t rows_a;      // valid extent of the UMMA-M slot
    int32_t rows_b;      // valid extent of the UMMA-N slot (the symbolic one for dense)
    int32_t n_full;      // UMMA N of full tiles
    int32_t n_tail;      // UMMA N of the last tile along the N slot (residue variant width)
    int32_t tiles_m;     // tile grid: tiles_m x tiles_n x batch
    int32_t tiles_n;
    int32_t batch;
    int32_t box_n;       // B rows (K-major) / columns (MN-major) per TMA stage; out/res box rows
    int32_t kb_total;    // ceil(K / 64)
    int32_t split;       // split-K factor (= cluster size along z); 1 -> persistent tile loop
    int32_t stages;      // smem pipeline depth
    int32_t a_batch_mid, b_batch_mid, out_batch_mid;   // tensor-map dim orders
    int32_t a_bcast, b_bcast;                          // broadcast batch (coordinate 0)
    int32_t a_static;    // 1: A (weights) is not written by in-flight kernels: TMA it before the PDL wait
    float alpha;
    void *out;
    int64_t ld_out;
    int64_t stride_out;
    const float *bias;
    const void *res;     // residual (split-K path reads it directly; otherwise via tmRes)
    int64_t ld_res;
    unsigned long long *trace;   // optional per-CTA phase timestamps (globaltimer ns), NULL = off
    int32_t dbg;                 // experiment bits (NIMBLE_DBG env): 1 skip split stores, 2 skip recv reads
    // device-resident extent (nimble_dense_dyn_dev): the symbolic token extent is read from
    // m_dev after the grid-dependency wait and the residue dispatch runs on the device;
    // rows_b / tiles_n / n_tail above then describe the upper bound M_max.
    const int32_t *m_dev;        // NULL = host extent
    int32_t var_c;               // variant limit c for the device dispatch
    CUtensorMap *out_slot;       // per-CTA global slots for the extent-patched output map
    nimble_dispatch *rec;        // optional device record of the device dispatch (CTA 0 writes it)
    // fused LayerNorm epilogue (EPI 4, pair family, rows of exactly 4 x 256 = 1024 features):
    // y = LN(acc + bias + res) * gamma + beta over each token's 1024 features.  The 8 CTAs of a
    // group (4 pairs = the 4 feature tiles of one token tile) exchange per-token partial sums
    // through ln_stats / ln_cnt (library workspace, counters self-resetting).
    const float *ln_gamma, *ln_beta;
    float ln_eps;
    int32_t ln_groups;           // groups of 4 pairs; pairs >= 4 * ln_groups idle
    float2 *ln_stats;            // [2 * ln_groups][8][256] (sum x, sum x^2) partials
    int32_t *ln_cnt;             // [2 * ln_groups][2] writers / readers per slot
    // half staging (2-CTA family, bf16, EPI <= 3): the epilogue stages and stores the tile in two
    // 128-token halves through a 32 KB buffer, which leaves room for a 6th pipeline stage
    int32_t half_stg;
    // k-blocks of 64 per pipeline stage: 2 where the operands are viewed as {64 k, rows, k-block}
    // (batch 1, K % 64 == 0; tensor maps tmA / tmB encoded that way), else 1
    int32_t kd;
};

struct UmmaLaunch {
    CUtensorMap tmA, tmB, tmOut, tmRes;
    UmmaParams p;
    dim3 grid;
    int b_mn_major, epi, out_f32, transposed;
    int pair;              // 1: 2-CTA clusters (tcgen05 cta_group::2, 256-row tiles)
    size_t smem_bytes;
    cudaStream_t stream;
};

cudaError_t launch_umma_gemm(const UmmaLaunch &L);
bool umma_static_available(int64_t M, int64_t N, int64_t K);
bool umma_static_bmm_available(int64_t M, int64_t N, int64_t K);
int umma_ln_max_groups(size_t smem_bytes);   // co-resident 4-pair groups for the fused-LN GEMM
cudaError_t launch_umma_gemm_static(const UmmaLaunch &L, int64_t M, int64_t N, int64_t K);
size_t umma_smem_bytes(int box_n, int b_mn_major, int stages, int split, int out_bytes, int transposed, int pair,
                       int half_stg, int kd);
// Programmatic dependent launch (griddepcontrol) on every libnimble launch that supports it.
bool pdl_enabled();

// Launch `kern` on `s` with the PDL attribute (when enabled).  Every kernel launched this
// way executes griddepcontrol.wait before touching memory written by earlier kernels.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
int umma_max_stages(int box_n, int b_mn_major, int kd);

// Weight-streaming dense (family 4, DISPATCH.md): few (feature tile, token tile) units, grid =
// S x m_tiles x n_tiles CTAs, the S K-splits of a unit one cluster; fp32 partial slabs reduced in
// split order via L2.
struct WsParams {
    int32_t M, N;            // tokens (symbolic), output features
    int32_t m_tiles, S;      // 128-feature tiles x K splits (cluster size S <= 16)
    int32_t n_tiles;         // 128-token tiles (the last one of width n_umma)
    int32_t kb_total;        // ceil(K / 64)
    int32_t n_umma;          // UMMA N of the last token tile (residue width, or 128 for the fallback)
    int32_t n_box;           // token rows per TMA box / partial slab row count
    int32_t stages;          // smem ring depth (weights of the first `stages` k-blocks prefetched)
    float alpha;
    const float *bias;
    const __nv_bfloat16 *res; int64_t ld_res;
    __nv_bfloat16 *out; int64_t ld_out;
    float *part;             // [n_tiles][m_tiles][S][n_box][128] fp32 partial slabs (workspace)
    // device-resident extent (nimble_dense_dyn_dev, one token tile): M is read from m_dev after
    // the grid-dependency wait, the residue dispatch (UMMA N of the tile) runs on the device and
    // CTA (0, 0) writes the record; M above is then the bound M_max
    const int32_t *m_dev;
    int32_t var_c;
    nimble_dispatch *rec;
    unsigned long long *trace;   // debug (nimble_debug_trace): per CTA 8 globaltimer stamps, NULL = off
};
struct WsLaunch {
    CUtensorMap tmA, tmB;    // W {K, N, 1} box {64, 128, 1}; x {K, M, 1} box {64, n_box, 1}
    WsParams p;
    int epi;                 // 0 alpha, 1 bias, 2 bias+GELU, 3 bias+residual
    size_t smem_bytes;
    cudaStream_t stream;
};
cudaError_t launch_ws_gemm(const WsLaunch &L);
size_t ws_smem_bytes(int n_box, int stages, int S);
bool ws_cluster_fits(int S, size_t smem_bytes);

// fp32 SIMT8 dense (family 0)
struct Simt8Params {
    const float *x; int64_t ldx;
    const float *W; int64_t ldw;
    const float *bias;
    const float *res; int64_t ldr;
    float *y; int64_t ldy;
    int32_t M, N, K, epi;
    int32_t k_tiles;      // k = floor(M / 8)
};
cudaError_t launch_simt8(const Simt8Params &p, int variant, dim3 grid, cudaStream_t s);
cudaError_t launch_simt8_static(const Simt8Params &p, dim3 grid, cudaStream_t s);   // M in 1..64

size_t attention_smem_bytes(int max_len);
int attention_max_requests();                     // R bound of one launch (work list in smem)
int attention_grid(int R, int max_len, int heads);   // persistent CTAs: <= 2 per SM
cudaError_t launch_attention_varlen(const CUtensorMap &tmQK, const CUtensorMap &tmV, const CUtensorMap &tmO,
                                    const CUtensorMap *tmOparts, const int32_t *seq_off,
                                    int R, int max_len, int heads, float scale, __nv_bfloat16 *out, int64_t ld_out,
                                    int64_t T_max, cudaStream_t s, CUtensorMap *map_slots, bool patch_T,
                                    unsigned long long *trace = nullptr);

cudaError_t launch_softmax_rows(const float *S, int64_t ldS, int64_t strideS, __nv_bfloat16 *P, int64_t ldP,
                                int64_t strideP, int64_t batch, int64_t rows, int64_t L, cudaStream_t s);
cudaError_t launch_layernorm(const __nv_bfloat16 *X, int64_t ldx, const float *g, const float *b, float eps,
                             __nv_bfloat16 *Y, int64_t ldy, int64_t rows, int64_t d, cudaStream_t s,
                             const int32_t *rows_dev = nullptr);

size_t lstm_workspace_bytes(int64_t H);
cudaError_t launch_lstm_seq(const float *G, int64_t ldg, const float *W_hh, int64_t ldw, const float *h0,
                            const float *c0, float *H_seq, int64_t ldh, float *hT, float *cT, int64_t T,
                            int64_t H, void *workspace, cudaStream_t s);

size_t lstm2_workspace_bytes(int64_t H);
// layer-1 input projection fused into the wavefront kernel (nimble_lstm2_forward)
struct Lstm2Input {
    const float *X; int64_t ldx;
    const float *Wih1; int64_t ldwi;
    const float *b1;
    int64_t I;
};
cudaError_t launch_lstm2_seq(const float *G1, int64_t ldg, const float *Whh1, const float *Wih2, const float *Whh2,
                             int64_t ldw, const float *b2, float *H1, float *H2, int64_t ldh, float *hT, float *cT,
                             int64_t T, int64_t H, void *workspace, cudaStream_t s,
                             const Lstm2Input *fused = nullptr);

struct TreeParams {
    const int32_t *nodes;
    const float *A; int64_t lda;
    const int32_t *a_rows;
    const float *W; int64_t ldw;
    const float *bias;
    const int32_t *parent_slot;
    float *hcat, *ccat; int64_t ldcat;
    float *h_out, *c_out; int64_t ldo;
    int32_t M, K, H, is_leaf;
};
cudaError_t launch_treelstm_level(const TreeParams &p, cudaStream_t s);

// Whole forest in one persistent launch: levels in height order, grid barrier between levels.
struct TreeForestParams {
    const float *X; int64_t ldx;            // word vectors (leaf inputs)
    const float *W_l, *b_l;                 // [3H x I], [3H]
    const float *U, *b_u;                   // [5H x 2H], [5H]
    const int32_t *level_off;               // [n_levels + 1], level 0 = leaves
    const int32_t *nodes, *rows, *pslot;    // [n_nodes] in level order
    float *hcat, *ccat; int64_t ldcat;
    float *h_out, *c_out; int64_t ldo;
    unsigned *counter;
    unsigned long long *trace;              // debug (nimble_debug_trace): [cta][level][2] stamps
    int32_t n_levels, I, H, max_level;
};
cudaError_t launch_treelstm_forest(const TreeForestParams &p, cudaStream_t s);

}  // namespace nimble
