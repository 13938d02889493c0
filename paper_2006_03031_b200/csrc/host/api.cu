// libnimble C ABI entry points (include/nimble.h): argument validation, the
// shape-function -> dispatch -> launch sequence of Nimble's InvokePacked path
// (App. A; §3.5 dispatch PAPER.md:387), TMA tensor-map
// encoding and asynchronous launches on the caller's stream.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../kernels/launch.h"
#include "internal.h"

namespace nimble {

static thread_local std::string t_err;
static thread_local nimble_dispatch t_last;
static thread_local bool t_has_last = false;

int fail(int status, const std::string &msg) {
    t_err = msg;
    return status;
}
void clear_error() { t_err.clear(); }
void record_dispatch(const nimble_dispatch &d) {
    t_last = d;
    t_has_last = true;
}

namespace {

int cuda_fail(const char *where, cudaError_t e) {
    return fail(NIMBLE_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- TMA encoding
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
cudaError_t g_encode_err = cudaSuccess;

cudaError_t get_encoder() {
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        g_encode_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (g_encode_err == cudaSuccess && (q != cudaDriverEntryPointSuccess || !fn))
            g_encode_err = cudaErrorNotSupported;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return g_encode_err;
}

// bf16 operand with inner (contiguous) dim `inner`, `rows` rows of stride `ld` elements,
// `batch` slices of stride `bstride` elements.  Dims are ordered by stride so heads that
// are interleaved inside a row (QKV views) become the middle dimension.
// box = {64 inner, box_rows rows, 1 slice}.  Returns whether batch is the middle dim.
int encode_operand(CUtensorMap *m, const void *base, int64_t inner, int64_t rows, int64_t ld, int64_t batch,
                   int64_t bstride, int box_rows, int *batch_mid) {
    cudaError_t e = get_encoder();
    if (e != cudaSuccess) return cuda_fail("cuTensorMapEncodeTiled lookup", e);
    cuuint64_t dims[3], strides[2];
    cuuint32_t box[3], estr[3] = {1, 1, 1};
    const bool mid = (batch > 1) && (bstride < ld);
    dims[0] = (cuuint64_t)inner;
    box[0] = 64;
    if (mid) {
        dims[1] = (cuuint64_t)batch; strides[0] = (cuuint64_t)bstride * 2; box[1] = 1;
        dims[2] = (cuuint64_t)rows;  strides[1] = (cuuint64_t)ld * 2;      box[2] = (cuuint32_t)box_rows;
    } else {
        dims[1] = (cuuint64_t)rows;  strides[0] = (cuuint64_t)ld * 2;      box[1] = (cuuint32_t)box_rows;
        dims[2] = (cuuint64_t)batch;
        strides[1] = (cuuint64_t)(batch > 1 ? bstride : ld * rows) * 2;
        box[2] = 1;
    }
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(NIMBLE_E_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
    *batch_mid = mid ? 1 : 0;
    return NIMBLE_OK;
}

// K-blocked operand view for two-k-block pipeline stages (batch 1, K % 64 == 0):
// dims {64 (k within a block), rows, K / 64 (k-block)}, strides {ld, 64 elements};
// box {64, box_rows, 2}: one TMA moves two consecutive swizzled 64-wide k-blocks.
int encode_operand_kb(CUtensorMap *m, const void *base, int64_t K, int64_t rows, int64_t ld, int box_rows, int kd = 2) {
    cudaError_t e = get_encoder();
    if (e != cudaSuccess) return cuda_fail("cuTensorMapEncodeTiled lookup", e);
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)kd}, estr[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(NIMBLE_E_CUDA, "cuTensorMapEncodeTiled(k-blocked) failed (code " + std::to_string((int)r) + ")");
    return NIMBLE_OK;
}

bool kblock2_enabled() {
    static const bool on = [] { const char *e = std::getenv("NIMBLE_KD"); return !(e && e[0] == '1'); }();
    return on;
}

// Output tile map for the transposed epilogue: out[b*bstride + j*ld + i], i < rows_i (inner),
// j < rows_j; box {128 i, box_j j, 1}, no swizzle.  TMA clips the box at the tensor bounds, so
// rows beyond the symbolic extent are never written.
int encode_out(CUtensorMap *m, void *base, bool f32, int64_t rows_i, int64_t rows_j, int64_t ld, int64_t batch,
               int64_t bstride, int box_j, int *batch_mid) {
    cudaError_t e = get_encoder();
    if (e != cudaSuccess) return cuda_fail("cuTensorMapEncodeTiled lookup", e);
    const int es = f32 ? 4 : 2;
    cuuint64_t dims[3], strides[2];
    cuuint32_t box[3], estr[3] = {1, 1, 1};
    const bool mid = (batch > 1) && (bstride < ld);
    dims[0] = (cuuint64_t)rows_i;
    // bf16 outputs / residuals: 64-feature boxes in the 128-B swizzle layout the kernel's
    // stmatrix / ldmatrix epilogue stages (two boxes per 128-feature tile); fp32: plain 128
    box[0] = f32 ? 128 : 64;
    if (mid) {
        dims[1] = (cuuint64_t)batch;  strides[0] = (cuuint64_t)bstride * es; box[1] = 1;
        dims[2] = (cuuint64_t)rows_j; strides[1] = (cuuint64_t)ld * es;      box[2] = (cuuint32_t)box_j;
    } else {
        dims[1] = (cuuint64_t)rows_j; strides[0] = (cuuint64_t)ld * es;      box[1] = (cuuint32_t)box_j;
        dims[2] = (cuuint64_t)batch;
        strides[1] = (cuuint64_t)(batch > 1 ? bstride : ld * rows_j) * es;
        box[2] = 1;
    }
    CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          f32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(NIMBLE_E_CUDA, "cuTensorMapEncodeTiled(out) failed (code " + std::to_string((int)r) + ")");
    *batch_mid = mid ? 1 : 0;
    return NIMBLE_OK;
}

bool ext_ok(int64_t x) { return x >= 1 && x <= kMaxExtent; }

// Fill the stage count / smem for a UMMA launch from the dispatch record.
// Pipeline depth / smem from the tile geometry, then the launch grid: the dispatch record's
// tile grid as is for split-K clusters, else min(tiles, 148) persistent CTAs.
unsigned long long *g_trace = nullptr;     // debug: per-CTA phase timestamps (nimble_debug_trace)
}  // namespace
unsigned long long *lstm_trace_buffer() { return g_trace; }
namespace {

void plan_pipeline(UmmaLaunch &L, const nimble_dispatch &d) {
    L.p.trace = g_trace;
    static const int dbg = [] { const char *e = std::getenv("NIMBLE_DBG"); return e ? std::atoi(e) : 0; }();
    L.p.dbg = dbg;
    if (L.p.kd < 1) L.p.kd = 1;
    const int kb_per_split = (L.p.kb_total + L.p.split - 1) / L.p.split;
    const int st_per_split = (kb_per_split + L.p.kd - 1) / L.p.kd;        // pipeline stages of kd k-blocks
    const int ob = L.out_f32 ? 4 : 2;
    static const int max_st = [] { const char *e = std::getenv("NIMBLE_MAX_STAGES"); return e ? std::atoi(e) : 8; }();
    int st = st_per_split < max_st ? st_per_split : max_st;     // NIMBLE_MAX_STAGES: experiment only
    if (st < 1) st = 1;
    // largest depth that fits next to the epilogue staging
    while (st > 1 && umma_smem_bytes(L.p.box_n, L.b_mn_major, st, L.p.split, ob, L.transposed, L.pair, L.p.half_stg,
                                     L.p.kd) > 232448)
        --st;
    L.p.stages = st;
    L.smem_bytes = umma_smem_bytes(L.p.box_n, L.b_mn_major, st, L.p.split, ob, L.transposed, L.pair, L.p.half_stg,
                                   L.p.kd);
    L.p.tiles_m = L.pair ? (L.p.rows_a + 255) / 256 : d.grid[0];   // pairs own 256-row tiles
    L.p.tiles_n = d.grid[1];
    L.p.batch = d.grid[2] / d.cluster[2];   // grid[2] = batch x cluster split-K
    const int64_t tiles = (int64_t)L.p.tiles_m * L.p.tiles_n * L.p.batch;
    const int64_t slots = L.pair ? kNumSMs / 2 : kNumSMs;
    if (L.p.split > 1) {
        L.grid = dim3(d.grid[0], d.grid[1], d.grid[2]);
    } else {
        const int64_t used = tiles < slots ? tiles : slots;
        L.grid = dim3((unsigned)(used * (L.pair ? 2 : 1)), 1, 1);
    }
}

}  // namespace
}  // namespace nimble

using namespace nimble;

extern "C" const char *nimble_last_error(void) { return t_err.c_str(); }

// Debug hook (not part of the product contract): when non-NULL, every subsequent tcgen05 GEMM
// launch writes 8 globaltimer stamps per CTA into buf[cta * 8 + slot].
extern "C" int nimble_debug_trace(unsigned long long *buf) {
    g_trace = buf;
    return NIMBLE_OK;
}
extern "C" const char *nimble_version(void) { return "nimble-b200 0.1 (sm_100a)"; }

extern "C" int nimble_last_dispatch(nimble_dispatch *out) {
    if (!out) return fail(NIMBLE_E_NULL, "nimble_last_dispatch: out is NULL");
    if (!t_has_last) return fail(NIMBLE_E_NULL, "nimble_last_dispatch: no launch yet on this thread");
    *out = t_last;
    return NIMBLE_OK;
}

// ------------------------------------------------------------------ dense_dyn
// Library workspace of the fused LayerNorm epilogue: per group of 4 CTA pairs, 2 slots of
// (sum, sum of squares) partials for 256 tokens x 8 CTAs, and 2 self-resetting counters per slot.
// One workspace per STREAM (a pool of kLnSlots per device, allocated together on the first fused
// launch of the device, so a stream first seen during graph capture needs no allocation): two
// streams running dense_ln_dyn concurrently never share counters.  More than kLnSlots distinct
// streams share slots round-robin (documented in include/nimble.h).
namespace nimble {
namespace {
constexpr int kLnMaxGroups = kNumSMs / 8;
constexpr int kLnSlots = 16;
constexpr size_t kLnStatsElems = (size_t)2 * kLnMaxGroups * 8 * 256;
constexpr size_t kLnCntElems = (size_t)2 * kLnMaxGroups * 2;
struct LnWorkspace {
    std::mutex mu;
    float2 *stats[64] = {};
    int32_t *cnt[64] = {};
    std::vector<std::pair<cudaStream_t, int>> owner[64];   // stream -> slot
};
LnWorkspace g_ln_ws;
cudaError_t ln_workspace(cudaStream_t stream, float2 **stats, int32_t **cnt) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_ln_ws.mu);
    if (!g_ln_ws.stats[dev]) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
            return cudaErrorStreamCaptureUnsupported;        // caller falls back to the two-launch form
        if ((e = cudaMalloc(&g_ln_ws.stats[dev], sizeof(float2) * kLnStatsElems * kLnSlots)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&g_ln_ws.cnt[dev], sizeof(int32_t) * kLnCntElems * kLnSlots)) != cudaSuccess) return e;
        if ((e = cudaMemset(g_ln_ws.cnt[dev], 0, sizeof(int32_t) * kLnCntElems * kLnSlots)) != cudaSuccess) return e;
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    }
    auto &own = g_ln_ws.owner[dev];
    int slot = -1;
    for (const auto &o : own)
        if (o.first == stream) slot = o.second;
    if (slot < 0) {
        slot = (int)(own.size() % kLnSlots);
        own.emplace_back(stream, slot);
    }
    *stats = g_ln_ws.stats[dev] + (size_t)slot * kLnStatsElems;
    *cnt = g_ln_ws.cnt[dev] + (size_t)slot * kLnCntElems;
    return cudaSuccess;
}
bool half_staging_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("NIMBLE_HALF_STG");
        return !(e && e[0] == '0');
    }();
    return on;
}
bool fused_ln_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("NIMBLE_FUSED_LN");
        return !(e && e[0] == '0');
    }();
    return on;
}
struct LnArgs {
    const float *gamma, *beta;
    float eps;
    bool fused;            // out: the LayerNorm ran in the GEMM epilogue
};
}  // namespace
}  // namespace nimble

// Library workspace of the weight-streaming family (4): per stream, the fp32 partial slabs of
// one launch (<= 148 CTAs x 128 tokens x 128 features).  Allocated when a stream is first seen
// (inside a graph capture the allocation runs in relaxed capture mode).  More than kWsSlots
// streams share slots round-robin (include/nimble.h: concurrent family-4 launches on streams
// that share a slot are not supported).
namespace nimble {
namespace {
constexpr int kWsSlots = 16;
constexpr size_t kWsPartElems = (size_t)kNumSMs * 128 * 128;   // <= 148 slabs (units x S <= 148)
struct WsWorkspace {
    std::mutex mu;
    std::vector<std::pair<cudaStream_t, int>> owner[64];
    float *part[64][kWsSlots] = {};
};
WsWorkspace g_ws;
cudaError_t ws_workspace(cudaStream_t stream, float **part) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    auto &own = g_ws.owner[dev];
    int slot = -1;
    for (const auto &o : own)
        if (o.first == stream) slot = o.second;
    if (slot < 0) {
        slot = (int)(own.size() % kWsSlots);
        own.emplace_back(stream, slot);
    }
    if (!g_ws.part[dev][slot]) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(stream, &cs)) != cudaSuccess) return e;
        const bool capturing = cs != cudaStreamCaptureStatusNone;
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        if (capturing) cudaThreadExchangeStreamCaptureMode(&mode);
        e = cudaMalloc(&g_ws.part[dev][slot], sizeof(float) * kWsPartElems);
        if (capturing) cudaThreadExchangeStreamCaptureMode(&mode);
        if (e != cudaSuccess) return e;
    }
    *part = g_ws.part[dev][slot];
    return cudaSuccess;
}

// Family 4 launch (DISPATCH.md): returns NIMBLE_OK, an error, or 1 when a cluster of S CTAs
// cannot be scheduled on this device (an SM partition smaller than the cluster under MPS /
// green contexts): the caller then takes family 1.
int launch_ws(const nimble_dispatch &d, const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
              const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N, int64_t K, int epi,
              cudaStream_t s, const int32_t *m_dev = nullptr, nimble_dispatch *rec = nullptr) {
    WsLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.p.M = (int32_t)M;
    L.p.N = (int32_t)N;
    L.p.m_tiles = d.grid[0];
    L.p.n_tiles = d.grid[1];
    L.p.S = d.split_k;
    L.p.kb_total = (int32_t)((K + 63) / 64);
    L.p.n_umma = d.r ? d.umma_n_tail : d.umma_n_full;
    L.p.n_box = d.grid[1] == 1 ? L.p.n_umma : d.umma_n_full;   // one box height for every token tile
    if (m_dev) L.p.n_box = d.umma_n_full;        // device extent: any residue width (incl. the fallback) fits
    const int kb_max = (L.p.kb_total + L.p.S - 1) / L.p.S;
    L.p.stages = kb_max < 3 ? kb_max : 3;
    L.smem_bytes = ws_smem_bytes(L.p.n_box, L.p.stages, L.p.S);
    static std::mutex fit_mu;
    static std::vector<std::pair<int, size_t>> fits;     // (S, smem) known to schedule
    {
        std::lock_guard<std::mutex> lk(fit_mu);
        bool known = false;
        for (const auto &f : fits) known |= (f.first == L.p.S && f.second == L.smem_bytes);
        if (!known) {
            if (!ws_cluster_fits(L.p.S, L.smem_bytes)) return 1;
            fits.emplace_back(L.p.S, L.smem_bytes);
        }
    }
    float *part = nullptr;
    cudaError_t e = ws_workspace(s, &part);
    if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn(family 4) workspace", e);
    L.p.part = part;
    L.p.trace = g_trace;
    L.p.m_dev = m_dev;                            // device extent: M above is the bound M_max
    L.p.var_c = variant_limit();
    L.p.rec = rec;
    L.p.alpha = 1.f;
    L.p.bias = bias;
    L.p.res = static_cast<const __nv_bfloat16 *>(residual);
    L.p.ld_res = ldr;
    L.p.out = static_cast<__nv_bfloat16 *>(y);
    L.p.ld_out = ldy;
    L.epi = epi;
    int st, mid = 0;
    if ((st = encode_operand(&L.tmA, W, K, N, ldw, 1, 0, 128, &mid)) != NIMBLE_OK) return st;
    if ((st = encode_operand(&L.tmB, x, K, M, ldx, 1, 0, L.p.n_box, &mid)) != NIMBLE_OK) return st;
    L.stream = s;
    e = launch_ws_gemm(L);
    if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn(family 4) launch", e);
    return NIMBLE_OK;
}
}  // namespace
}  // namespace nimble

static int dense_impl(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                      const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N,
                      int64_t K, int dt, int epi, void *stream, bool static_twin, LnArgs *ln = nullptr) {
    // 1. shape function (runtime type-relation check)
    const int64_t xs[2] = {M, K}, ws[2] = {N, K};
    int64_t os[2];
    if (!ext_ok(M) || !ext_ok(N) || !ext_ok(K)) return fail(NIMBLE_E_EXTENT, "nimble_dense_dyn: extents must be in [1, 2^31-1]");
    int st = nimble_shape_dense(xs, ws, os);
    if (st != NIMBLE_OK) return st;
    if (!x || !W || !y) return fail(NIMBLE_E_NULL, "nimble_dense_dyn: x, W and y must be non-NULL");
    if (epi < NIMBLE_EPI_NONE || epi > NIMBLE_EPI_BIAS_RESIDUAL) return fail(NIMBLE_E_DTYPE, "nimble_dense_dyn: unknown epilogue");
    if (epi >= NIMBLE_EPI_BIAS && !bias) return fail(NIMBLE_E_NULL, "nimble_dense_dyn: bias required by the epilogue");
    if (epi == NIMBLE_EPI_BIAS_RESIDUAL && !residual) return fail(NIMBLE_E_NULL, "nimble_dense_dyn: residual required");
    if (ldx < K || ldw < K || ldy < N || (epi == NIMBLE_EPI_BIAS_RESIDUAL && ldr < N))
        return fail(NIMBLE_E_SHAPE, "nimble_dense_dyn: leading dimension smaller than the row length");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    nimble_dispatch d;

    if (dt == NIMBLE_F32) {
        if (!aligned16(x) || !aligned16(W) || ldx % 4 || ldw % 4 || K % 4)
            return fail(NIMBLE_E_ALIGN, "nimble_dense_dyn(f32): x/W need 16-B alignment, ldx, ldw, K multiples of 4");
        dispatch_simt8(M, N, &d);                     // 2. dispatch by residue
        Simt8Params p{static_cast<const float *>(x), ldx, static_cast<const float *>(W), ldw, bias,
                      static_cast<const float *>(residual), ldr, static_cast<float *>(y), ldy,
                      (int32_t)M, (int32_t)N, (int32_t)K, epi, (int32_t)d.k};
        if (static_twin && M > 64) return fail(NIMBLE_E_UNSUPPORTED, "nimble_dense_static(f32): M must be in 1..64");
        cudaError_t e = static_twin ? launch_simt8_static(p, dim3(d.grid[0], d.grid[1], d.grid[2]), s)
                                    : launch_simt8(p, d.variant, dim3(d.grid[0], d.grid[1], d.grid[2]), s);
        if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn(f32) launch", e);
        record_dispatch(d);
        clear_error();
        return NIMBLE_OK;
    }
    if (dt != NIMBLE_BF16) return fail(NIMBLE_E_DTYPE, "nimble_dense_dyn: unknown dtype");
    if (!aligned16(x) || !aligned16(W) || !aligned16(y) || ((ldx * 2) % 16) || ((ldw * 2) % 16) || ((ldy * 2) % 16) ||
        (epi == NIMBLE_EPI_BIAS_RESIDUAL && (!aligned16(residual) || (ldr * 2) % 16)))
        return fail(NIMBLE_E_ALIGN, "nimble_dense_dyn(bf16): TMA needs 16-B aligned x/W/y/residual and ld*2 % 16 == 0");
    if (static_twin) dispatch_umma_t(1, M, N, K, &d);   // static twins are compiled for family 1/3, t = 128
    else dispatch_dense_bf16(M, N, K, &d);               // tuned schedule, if registered; family 4 at M <= 128
    if (d.family == 4) {
        // (dense_ln_dyn: the LayerNorm needs whole rows across feature tiles, i.e. across
        // clusters: it stays a separate launch after the family-4 GEMM)
        const int ws = launch_ws(d, x, ldx, W, ldw, bias, residual, ldr, y, ldy, M, N, K, epi, s);
        if (ws == NIMBLE_OK) {
            record_dispatch(d);
            clear_error();
            return NIMBLE_OK;
        }
        if (ws != 1) return ws;
        int32_t t = 0, cap = 8;                      // not co-resident here: family 1
        dense_schedule(N, K, &t, &cap);
        dispatch_umma_t(1, M, N, K, &d, t, cap);
    }
    UmmaLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.b_mn_major = 0;
    L.p.rows_a = (int32_t)N;             // weights on the UMMA-M slot
    L.p.rows_b = (int32_t)M;             // tokens on the UMMA-N slot (symbolic)
    L.p.n_full = d.umma_n_full;
    L.p.n_tail = d.r ? d.umma_n_tail : d.umma_n_full;
    L.p.box_n = (d.grid[1] == 1) ? L.p.n_tail : d.umma_n_full;
    L.p.kb_total = (int32_t)((K + 63) / 64);
    L.p.split = d.cluster[2];            // cluster split-K (1: none; a stream-K tail is planned separately)
    L.epi = epi;
    L.out_f32 = 0;
    L.transposed = 1;
    L.p.alpha = 1.f;
    L.p.out = y;
    L.p.ld_out = ldy;
    L.p.stride_out = 0;
    L.p.bias = bias;
    L.p.res = residual;
    L.p.ld_res = ldr;
    L.p.a_static = pdl_enabled() ? 1 : 0;   // weights: fetched before the PDL grid-dependency wait
    L.pair = (d.family == 3) ? 1 : 0;       // large M: 2-CTA pairs, each CTA loads half of B
    const int box_b = L.pair ? L.p.box_n / 2 : L.p.box_n;
    // LayerNorm fusion (nimble_dense_ln_dyn): fused only where a group of 4 pairs covers the
    // whole row (family 3, N = 4 x 256) and the main loop is long enough (K >= 2048) to hide the
    // epilogue's cross-CTA exchange; at K = 1024 (BERT's O-projection) the fused epilogue
    // costs what the LN launch saves
    bool ln_fused = false;
    if (ln) {
        const char *mk = std::getenv("NIMBLE_LN_MIN_K");      // experiment knob (default 2048)
        const int64_t min_k = mk ? std::atoll(mk) : 2048;
        ln_fused = fused_ln_enabled() && L.pair && N == 1024 && K >= min_k && epi == NIMBLE_EPI_BIAS_RESIDUAL &&
                   !static_twin;
    }
    // the 2-CTA family stages its bf16 output in 128-token halves (a third 64 KB pipeline stage
    // fits); the fused LayerNorm then normalises each half (tokens are independent rows)
    L.p.half_stg = (L.pair && half_staging_enabled()) ? 1 : 0;
    const int out_box = L.p.half_stg ? L.p.box_n / 2 : L.p.box_n;
    // two k-blocks per pipeline stage where the operands tile K exactly (every BERT shape)
    L.p.kd = (kblock2_enabled() && K % 64 == 0 && K >= 128) ? 2 : 1;
    // (the second session took kd = 3 for the 1-CTA family without split-K, 2-7 % faster with
    // the lane-0 MMA issuer; with the converged-warp issuer kd = 2 is 0-5 % faster at every
    // family-1 point, profiles/r02e_kd_ab.jsonl, so every family streams kd = 2 again)
    static const int kd_exp = [] { const char *e = std::getenv("NIMBLE_EXP_KD"); return e ? std::atoi(e) : 0; }();
    if (kd_exp >= 2 && L.p.kd >= 2) L.p.kd = kd_exp;   // experiment only: k-blocks per stage
    if (L.p.kd >= 2) {
        if ((st = encode_operand_kb(&L.tmA, W, K, N, ldw, 128, L.p.kd)) != NIMBLE_OK) return st;
        if ((st = encode_operand_kb(&L.tmB, x, K, M, ldx, box_b, L.p.kd)) != NIMBLE_OK) return st;
    } else {
        if ((st = encode_operand(&L.tmA, W, K, N, ldw, 1, 0, 128, &L.p.a_batch_mid)) != NIMBLE_OK) return st;
        if ((st = encode_operand(&L.tmB, x, K, M, ldx, 1, 0, box_b, &L.p.b_batch_mid)) != NIMBLE_OK) return st;
    }
    if ((st = encode_out(&L.tmOut, y, false, N, M, ldy, 1, 0, out_box, &L.p.out_batch_mid)) != NIMBLE_OK) return st;
    if (epi == NIMBLE_EPI_BIAS_RESIDUAL) {
        int mid = 0;
        if ((st = encode_out(&L.tmRes, const_cast<void *>(residual), false, N, M, ldr, 1, 0, out_box, &mid)) != NIMBLE_OK) return st;
    } else {
        L.tmRes = L.tmOut;
    }
    L.p.box_n = box_b;
    if (L.pair && (L.p.a_batch_mid || L.p.b_batch_mid || L.p.out_batch_mid))
        return fail(NIMBLE_E_UNSUPPORTED, "nimble_dense_dyn: dense operands are single-batch (internal error)");
    plan_pipeline(L, d);
    L.stream = s;
    if (ln) {
        // the 8 CTAs of a group spin on each other: every group must be co-resident, so the
        // group count is capped by the occupancy API's count of co-resident CTA pairs (fewer
        // SMs under MPS / green contexts shrink it; none left -> the two-launch form)
        const int max_groups = ln_fused ? umma_ln_max_groups(L.smem_bytes) : 0;
        if (max_groups < 1) ln_fused = false;
        if (ln_fused && ln_workspace(s, &L.p.ln_stats, &L.p.ln_cnt) != cudaSuccess) {
            cudaGetLastError();
            ln_fused = false;                                   // e.g. first use inside a capture
        }
        ln->fused = ln_fused;
        if (ln->fused) {
            int groups = L.p.tiles_n < kLnMaxGroups ? L.p.tiles_n : kLnMaxGroups;
            if (groups > max_groups) groups = max_groups;
            L.p.ln_groups = groups;
            L.p.ln_gamma = ln->gamma;
            L.p.ln_beta = ln->beta;
            L.p.ln_eps = ln->eps;
            L.grid = dim3((unsigned)(8 * groups), 1, 1);
            L.epi = 4;
        }
    }
    if (static_twin && (epi != NIMBLE_EPI_BIAS || !umma_static_available(M, N, K)))
        return fail(NIMBLE_E_UNSUPPORTED, "nimble_dense_static(bf16): (M, N, K) not compiled in, or epilogue != BIAS");
    cudaError_t e = static_twin ? launch_umma_gemm_static(L, M, N, K) : launch_umma_gemm(L);
    if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn(bf16) launch", e);
    record_dispatch(d);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_dense_dyn(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                                const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N,
                                int64_t K, int dt, int epi, void *stream) {
    return dense_impl(x, ldx, W, ldw, bias, residual, ldr, y, ldy, M, N, K, dt, epi, stream, false);
}

extern "C" int nimble_dense_ln_dyn(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                                   const void *residual, int64_t ldr, const float *gamma, const float *beta, float eps,
                                   void *y, int64_t ldy, int64_t M, int64_t N, int64_t K, void *stream) {
    if (!gamma || !beta || !bias || !residual) return fail(NIMBLE_E_NULL, "nimble_dense_ln_dyn: bias, residual, gamma, beta required");
    if (!aligned16(gamma) || !aligned16(beta)) return fail(NIMBLE_E_ALIGN, "nimble_dense_ln_dyn: gamma / beta 16-B aligned");
    if (N > 4096 || N % 8) return fail(NIMBLE_E_UNSUPPORTED, "nimble_dense_ln_dyn: N must be a multiple of 8, <= 4096");
    LnArgs ln{gamma, beta, eps, false};
    int st = dense_impl(x, ldx, W, ldw, bias, residual, ldr, y, ldy, M, N, K, NIMBLE_BF16, NIMBLE_EPI_BIAS_RESIDUAL,
                        stream, false, &ln);
    if (st != NIMBLE_OK || ln.fused) return st;
    // not fusable at this (M, N): the same two steps as separate launches, LayerNorm in place
    nimble_dispatch keep = t_last;
    static const bool skip_ln = [] { const char *e = std::getenv("NIMBLE_EXP_SKIP_LN"); return e && e[0] == '1'; }();
    if (skip_ln) return NIMBLE_OK;           // experiment only (timing of the LayerNorm launch): wrong results
    st = nimble_layernorm(y, ldy, gamma, beta, eps, y, ldy, M, N, stream);
    t_last = keep;
    return st;
}

extern "C" int nimble_dense_static(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                                   const void *residual, int64_t ldr, void *y, int64_t ldy, int64_t M, int64_t N,
                                   int64_t K, int dt, int epi, void *stream) {
    return dense_impl(x, ldx, W, ldw, bias, residual, ldr, y, ldy, M, N, K, dt, epi, stream, true);
}

// ------------------------------------------------------------------ dense_dyn_dev
namespace nimble {
namespace {
// Library-owned ring of per-CTA tensor-map slots for device-extent launches: launch i uses
// block i % kSlotRing, so a kernel never patches a slot an in-flight neighbour still reads
// (PDL overlaps adjacent kernels only).  One ring per device, allocated on first use.
constexpr int kSlotRing = 64;
struct SlotRing {
    int per_launch;                       // maps per launch block
    std::mutex mu;
    CUtensorMap *buf[64] = {};            // per device
    std::atomic<uint32_t> seq{0};
};
SlotRing g_gemm_slots{kNumSMs};           // one output map per persistent CTA
SlotRing g_attn_slots{2 * 2 * kNumSMs};   // Q/K and V maps per persistent CTA (<= 2 per SM)

cudaError_t next_slot_block(SlotRing &ring, CUtensorMap **out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    {
        std::lock_guard<std::mutex> lk(ring.mu);
        if (!ring.buf[dev]) {
            e = cudaMalloc(&ring.buf[dev], sizeof(CUtensorMap) * (size_t)kSlotRing * ring.per_launch);
            if (e != cudaSuccess) return e;
        }
    }
    *out = ring.buf[dev] + (size_t)(ring.seq.fetch_add(1) % kSlotRing) * ring.per_launch;
    return cudaSuccess;
}
}  // namespace
}  // namespace nimble

extern "C" int nimble_dense_dyn_dev(const void *x, int64_t ldx, const void *W, int64_t ldw, const float *bias,
                                    const void *residual, int64_t ldr, void *y, int64_t ldy, const int32_t *M_dev,
                                    int64_t M_max, int64_t N, int64_t K, int epi, nimble_dispatch *dispatch_dev,
                                    void *stream) {
    if (!ext_ok(M_max) || !ext_ok(N) || !ext_ok(K)) return fail(NIMBLE_E_EXTENT, "nimble_dense_dyn_dev: extents must be in [1, 2^31-1]");
    if (M_max >= 2048) return fail(NIMBLE_E_UNSUPPORTED, "nimble_dense_dyn_dev: M_max must be < 2048 (family 1)");
    const int64_t xs[2] = {M_max, K}, ws[2] = {N, K};
    int64_t os[2];
    int st = nimble_shape_dense(xs, ws, os);           // upper-bound shape
    if (st != NIMBLE_OK) return st;
    if (!x || !W || !y || !M_dev) return fail(NIMBLE_E_NULL, "nimble_dense_dyn_dev: x, W, y and M_dev must be non-NULL");
    if (epi < NIMBLE_EPI_NONE || epi > NIMBLE_EPI_BIAS_RESIDUAL) return fail(NIMBLE_E_DTYPE, "nimble_dense_dyn_dev: unknown epilogue");
    if (epi >= NIMBLE_EPI_BIAS && !bias) return fail(NIMBLE_E_NULL, "nimble_dense_dyn_dev: bias required by the epilogue");
    if (epi == NIMBLE_EPI_BIAS_RESIDUAL && !residual) return fail(NIMBLE_E_NULL, "nimble_dense_dyn_dev: residual required");
    if (ldx < K || ldw < K || ldy < N || (epi == NIMBLE_EPI_BIAS_RESIDUAL && ldr < N))
        return fail(NIMBLE_E_SHAPE, "nimble_dense_dyn_dev: leading dimension smaller than the row length");
    if (!aligned16(x) || !aligned16(W) || !aligned16(y) || ((ldx * 2) % 16) || ((ldw * 2) % 16) || ((ldy * 2) % 16) ||
        (epi == NIMBLE_EPI_BIAS_RESIDUAL && (!aligned16(residual) || (ldr * 2) % 16)))
        return fail(NIMBLE_E_ALIGN, "nimble_dense_dyn_dev: TMA needs 16-B aligned x/W/y/residual and ld*2 % 16 == 0");
    int32_t t = 0, cap = 8;
    dense_schedule(N, K, &t, &cap);                    // tuned token tile / split cap
    nimble_dispatch d;
    if (t == 0 && M_max <= 128 && (N + 127) / 128 <= kNumSMs) {
        // family 4 (one token tile): the split S depends on (N, K) only, so the launch geometry of
        // the bound serves every M <= M_max; the kernel reads M and picks the residue width
        dispatch_umma_ws(M_max, N, K, &d);
        const int ws = launch_ws(d, x, ldx, W, ldw, bias, residual, ldr, y, ldy, M_max, N, K, epi,
                                 static_cast<cudaStream_t>(stream), M_dev, dispatch_dev);
        if (ws == NIMBLE_OK) {
            clear_error();
            return NIMBLE_OK;
        }
        if (ws != 1) return ws;
    }
    // split-K needs a launch grid that does not depend on M: allowed when the bound fits ONE
    // token tile, where the host rule's split (a function of the tile count) is the same for
    // every M <= M_max; otherwise the device dispatch runs split 1
    dispatch_umma_t(1, M_max, N, K, &d, t, cap);        // t = 0: the default rule (t = 128, K-dependent cap)
    // (family 3, which the wave rule can pick for a wide N, has no device-side geometry: the
    // device path runs family 1 at t = 128 then too)
    if (d.grid[1] != 1 || d.family == 3) dispatch_umma_t(1, M_max, N, K, &d, t > 0 ? t : 128, 1);   // geometry for the bound
    UmmaLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.p.rows_a = (int32_t)N;
    L.p.rows_b = (int32_t)M_max;
    L.p.n_full = d.umma_n_full;
    L.p.n_tail = d.r ? d.umma_n_tail : d.umma_n_full;
    L.p.box_n = d.umma_n_full;                         // fixed box: the tail width is decided on device
    L.p.kb_total = (int32_t)((K + 63) / 64);
    L.p.split = d.cluster[2];            // cluster split-K (1: none; a stream-K tail is planned separately)
    L.epi = epi;
    L.transposed = 1;
    L.p.alpha = 1.f;
    L.p.out = y;
    L.p.ld_out = ldy;
    L.p.bias = bias;
    L.p.res = residual;
    L.p.ld_res = ldr;
    L.p.a_static = pdl_enabled() ? 1 : 0;
    L.p.m_dev = M_dev;
    L.p.var_c = variant_limit();
    L.p.rec = dispatch_dev;
    L.p.kd = (kblock2_enabled() && K % 64 == 0 && K >= 128) ? 2 : 1;
    if (L.p.kd == 2 && L.p.split == 1 && K >= 192) L.p.kd = 3;   // as dense_impl's 1-CTA family
    if (L.p.kd >= 2) {
        if ((st = encode_operand_kb(&L.tmA, W, K, N, ldw, 128, L.p.kd)) != NIMBLE_OK) return st;
        if ((st = encode_operand_kb(&L.tmB, x, K, M_max, ldx, L.p.box_n, L.p.kd)) != NIMBLE_OK) return st;
    } else {
        if ((st = encode_operand(&L.tmA, W, K, N, ldw, 1, 0, 128, &L.p.a_batch_mid)) != NIMBLE_OK) return st;
        if ((st = encode_operand(&L.tmB, x, K, M_max, ldx, 1, 0, L.p.box_n, &L.p.b_batch_mid)) != NIMBLE_OK) return st;
    }
    if ((st = encode_out(&L.tmOut, y, false, N, M_max, ldy, 1, 0, L.p.box_n, &L.p.out_batch_mid)) != NIMBLE_OK) return st;
    if (epi == NIMBLE_EPI_BIAS_RESIDUAL) {
        int mid = 0;
        if ((st = encode_out(&L.tmRes, const_cast<void *>(residual), false, N, M_max, ldr, 1, 0, L.p.box_n, &mid)) != NIMBLE_OK) return st;
    } else {
        L.tmRes = L.tmOut;
    }
    cudaError_t e = next_slot_block(g_gemm_slots, &L.p.out_slot);
    if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn_dev slot ring", e);
    plan_pipeline(L, d);
    L.stream = static_cast<cudaStream_t>(stream);
    e = launch_umma_gemm(L);
    if (e != cudaSuccess) return cuda_fail("nimble_dense_dyn_dev launch", e);
    clear_error();
    return NIMBLE_OK;
}

// ------------------------------------------------------------------ bmm_dyn
static int bmm_impl(const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                    int64_t strideB, int trans_b, void *Cout, int64_t ldc, int64_t strideC, int64_t batch,
                    int64_t M, int64_t N, int64_t K, float alpha, int in_dt, int out_dt, void *stream,
                    bool static_twin) {
    if (!ext_ok(batch) || !ext_ok(M) || !ext_ok(N) || !ext_ok(K))
        return fail(NIMBLE_E_EXTENT, "nimble_bmm_dyn: extents must be in [1, 2^31-1]");
    const int64_t as[3] = {batch, M, K};
    const int64_t bs[3] = {batch, trans_b ? K : N, trans_b ? N : K};
    int64_t os[3];
    int st = nimble_shape_bmm(as, bs, trans_b, os);
    if (st != NIMBLE_OK) return st;
    if (!A || !B || !Cout) return fail(NIMBLE_E_NULL, "nimble_bmm_dyn: A, B and C must be non-NULL");
    if (in_dt == NIMBLE_F32) return fail(NIMBLE_E_UNSUPPORTED, "nimble_bmm_dyn: fp32 inputs are not built (bf16 only)");
    if (in_dt != NIMBLE_BF16 || (out_dt != NIMBLE_BF16 && out_dt != NIMBLE_F32))
        return fail(NIMBLE_E_DTYPE, "nimble_bmm_dyn: unknown dtype");
    if (lda < K || ldb < (trans_b ? N : K) || ldc < N) return fail(NIMBLE_E_SHAPE, "nimble_bmm_dyn: leading dimension too small");
    const int osz = out_dt == NIMBLE_F32 ? 4 : 2;
    if (!aligned16(A) || !aligned16(B) || !aligned16(Cout) || (lda * 2) % 16 || (ldb * 2) % 16 ||
        (strideA * 2) % 16 || (strideB * 2) % 16 || (ldc * osz) % 16 || (strideC * osz) % 16)
        return fail(NIMBLE_E_ALIGN, "nimble_bmm_dyn: bases, leading dims and batch strides must be 16-B multiples");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    nimble_dispatch d;
    nimble_dispatch_bmm(batch, M, N, K, trans_b, in_dt, &d);
    UmmaLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.p.kb_total = (int32_t)((K + 63) / 64);
    L.p.split = d.cluster[2];            // cluster split-K (1: none; a stream-K tail is planned separately)
    L.epi = 0;
    L.out_f32 = out_dt == NIMBLE_F32;
    L.p.alpha = alpha;
    L.p.out = Cout;
    L.p.ld_out = ldc;
    L.p.stride_out = strideC;
    L.p.n_full = d.umma_n_full;
    if (!trans_b) {
        // family 1: B rows (N) on the UMMA-M slot, A rows (M, symbolic) on the UMMA-N slot
        L.b_mn_major = 0;
        L.p.rows_a = (int32_t)N;
        L.p.rows_b = (int32_t)M;
        L.p.n_tail = d.r ? d.umma_n_tail : d.umma_n_full;
        L.p.box_n = (d.grid[1] == 1) ? L.p.n_tail : d.umma_n_full;
        L.transposed = 1;
        L.pair = (d.family == 3) ? 1 : 0;
        const int box_b = L.pair ? L.p.box_n / 2 : L.p.box_n;
        if ((st = encode_operand(&L.tmA, B, K, N, ldb, batch, strideB, 128, &L.p.a_batch_mid)) != NIMBLE_OK) return st;
        if ((st = encode_operand(&L.tmB, A, K, M, lda, batch, strideA, box_b, &L.p.b_batch_mid)) != NIMBLE_OK) return st;
        if ((st = encode_out(&L.tmOut, Cout, out_dt == NIMBLE_F32, N, M, ldc, batch, strideC, L.p.box_n,
                             &L.p.out_batch_mid)) != NIMBLE_OK) return st;
        L.tmRes = L.tmOut;
        L.p.box_n = box_b;
    } else {
        // family 2: A rows (M) on the UMMA-M slot, columns of B (N) MN-major on the UMMA-N slot
        L.b_mn_major = 1;
        L.p.rows_a = (int32_t)M;
        L.p.rows_b = (int32_t)N;
        L.p.n_tail = d.umma_n_tail;
        L.p.box_n = d.umma_n_full;
        L.transposed = 0;
        if ((st = encode_operand(&L.tmA, A, K, M, lda, batch, strideA, 128, &L.p.a_batch_mid)) != NIMBLE_OK) return st;
        // B is [K x N]: inner dim N (contiguous), K rows; box {64 cols, 64 k-rows}
        if ((st = encode_operand(&L.tmB, B, N, K, ldb, batch, strideB, 64, &L.p.b_batch_mid)) != NIMBLE_OK) return st;
        L.tmOut = L.tmA;                      // unused by the direct epilogue
        L.tmRes = L.tmA;
    }
    plan_pipeline(L, d);
    L.stream = s;
    if (static_twin && (trans_b || out_dt != NIMBLE_F32 || !umma_static_bmm_available(M, N, K)))
        return fail(NIMBLE_E_UNSUPPORTED, "nimble_bmm_static: (M, N, K) not compiled in, or trans_b / bf16 output");
    cudaError_t e = static_twin ? launch_umma_gemm_static(L, M, N, K) : launch_umma_gemm(L);
    if (e != cudaSuccess) return cuda_fail("nimble_bmm_dyn launch", e);
    record_dispatch(d);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_bmm_dyn(const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                              int64_t strideB, int trans_b, void *Cout, int64_t ldc, int64_t strideC, int64_t batch,
                              int64_t M, int64_t N, int64_t K, float alpha, int in_dt, int out_dt, void *stream) {
    return bmm_impl(A, lda, strideA, B, ldb, strideB, trans_b, Cout, ldc, strideC, batch, M, N, K, alpha, in_dt,
                    out_dt, stream, false);
}

extern "C" int nimble_bmm_static(const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                                 int64_t strideB, int trans_b, void *Cout, int64_t ldc, int64_t strideC, int64_t batch,
                                 int64_t M, int64_t N, int64_t K, float alpha, int in_dt, int out_dt, void *stream) {
    return bmm_impl(A, lda, strideA, B, ldb, strideB, trans_b, Cout, ldc, strideC, batch, M, N, K, alpha, in_dt,
                    out_dt, stream, true);
}

// ------------------------------------------------------------------ varlen attention
static int attention_impl(const void *qkv, int64_t ld_qkv, int64_t T, const int32_t *seq_off, int32_t R,
                                       int32_t max_len, int32_t heads, int32_t head_dim, float scale, void *out,
                                       int64_t ld_out, void *stream, bool dev) {
    if (!qkv || !seq_off || !out) return fail(NIMBLE_E_NULL, "nimble_attention_varlen: NULL pointer");
    if (!ext_ok(T) || R < 1 || max_len < 1 || heads < 1 || head_dim < 1)
        return fail(NIMBLE_E_EXTENT, "nimble_attention_varlen: extents must be >= 1");
    if (head_dim != 64) return fail(NIMBLE_E_UNSUPPORTED, "nimble_attention_varlen: head_dim must be 64");
    if (max_len > 8192) return fail(NIMBLE_E_UNSUPPORTED, "nimble_attention_varlen: max_len > 8192 not built");

    if (ld_qkv < 3LL * heads * head_dim || ld_out < (int64_t)heads * head_dim)
        return fail(NIMBLE_E_SHAPE, "nimble_attention_varlen: leading dimension too small");
    if (!aligned16(qkv) || !aligned16(out) || (ld_qkv * 2) % 16 || (ld_out * 2) % 16)
        return fail(NIMBLE_E_ALIGN, "nimble_attention_varlen: 16-B aligned qkv/out and ld*2 % 16 == 0 required");
    cudaError_t e = get_encoder();
    if (e != cudaSuccess) return cuda_fail("cuTensorMapEncodeTiled lookup", e);
    // packed QKV viewed as {64 (e), 3*heads (Q heads | K heads | V heads), T (tokens)}
    CUtensorMap tmQK, tmV;
    cuuint64_t dims[3] = {64, (cuuint64_t)(3 * heads), (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)head_dim * 2, (cuuint64_t)ld_qkv * 2};
    cuuint32_t estr[3] = {1, 1, 1};
    cuuint32_t box_qk[3] = {64, 1, 128}, box_v[3] = {64, 1, 64};
    CUresult r = g_encode(&tmQK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(qkv), dims, strides, box_qk,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
        r = g_encode(&tmV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(qkv), dims, strides, box_v, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    // output [T x ld_out] bf16: 2-D view {heads * 64 columns, T rows}, box {64, 128} in the
    // 128-B swizzle the kernel stages full query tiles in (one TMA store per full tile)
    // (+ the same view with 64 / 32 / 16 / 8-row boxes for the valid rows of partial tiles)
    CUtensorMap tmO, tmOp[4];
    for (int b = -1; b < 4 && r == CUDA_SUCCESS; ++b) {
        cuuint64_t odims[2] = {(cuuint64_t)heads * 64, (cuuint64_t)T};
        cuuint64_t ostr[1] = {(cuuint64_t)ld_out * 2};
        cuuint32_t obox[2] = {64, b < 0 ? 128u : (64u >> b)}, oestr[2] = {1, 1};
        r = g_encode(b < 0 ? &tmO : &tmOp[b], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, odims, ostr, obox, oestr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return fail(NIMBLE_E_CUDA, "cuTensorMapEncodeTiled(attention) failed (code " + std::to_string((int)r) + ")");
    // per-CTA tensor-map slots: the device-extent form patches its Q/K and V maps (extent T)
    CUtensorMap *slots = nullptr;
    if (dev) {
        e = next_slot_block(g_attn_slots, &slots);
        if (e != cudaSuccess) return cuda_fail("nimble_attention_varlen_dev slot ring", e);
    }
    // the kernel's work list holds attention_max_requests() requests: longer streams run as
    // consecutive launches over request chunks (seq_off entries are absolute token offsets, so a
    // chunk is just a shifted seq_off pointer; the device-extent form reads its chunk's end)
    const int chunk = attention_max_requests();
    for (int32_t r0 = 0; r0 < R; r0 += chunk) {
        const int32_t Rc = R - r0 < chunk ? R - r0 : chunk;
        CUtensorMap *sl = slots;
        if (dev && r0 > 0) {
            e = next_slot_block(g_attn_slots, &sl);
            if (e != cudaSuccess) return cuda_fail("nimble_attention_varlen_dev slot ring", e);
        }
        e = launch_attention_varlen(tmQK, tmV, tmO, tmOp, seq_off + r0, Rc, max_len, heads, scale,
                                    static_cast<__nv_bfloat16 *>(out), ld_out, T, static_cast<cudaStream_t>(stream), sl,
                                    dev, g_trace);
        if (e != cudaSuccess) return cuda_fail("nimble_attention_varlen launch", e);
    }
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_attention_varlen(const void *qkv, int64_t ld_qkv, int64_t T, const int32_t *seq_off, int32_t R,
                                       int32_t max_len, int32_t heads, int32_t head_dim, float scale, void *out,
                                       int64_t ld_out, void *stream) {
    return attention_impl(qkv, ld_qkv, T, seq_off, R, max_len, heads, head_dim, scale, out, ld_out, stream, false);
}

extern "C" int nimble_attention_varlen_dev(const void *qkv, int64_t ld_qkv, int64_t T_max, const int32_t *seq_off,
                                           int32_t R, int32_t max_len, int32_t heads, int32_t head_dim, float scale,
                                           void *out, int64_t ld_out, void *stream) {
    return attention_impl(qkv, ld_qkv, T_max, seq_off, R, max_len, heads, head_dim, scale, out, ld_out, stream, true);
}

// ------------------------------------------------------------------ row ops
extern "C" int nimble_softmax_rows(const float *S, int64_t ldS, int64_t strideS, void *P, int64_t ldP, int64_t strideP,
                                   int64_t batch, int64_t rows, int64_t L, void *stream) {
    if (!S || !P) return fail(NIMBLE_E_NULL, "nimble_softmax_rows: NULL pointer");
    if (!ext_ok(batch) || !ext_ok(rows) || !ext_ok(L)) return fail(NIMBLE_E_EXTENT, "nimble_softmax_rows: extents must be >= 1");
    if (ldS < L || ldP < L) return fail(NIMBLE_E_SHAPE, "nimble_softmax_rows: ld < L");
    if (L > 1024) return fail(NIMBLE_E_UNSUPPORTED, "nimble_softmax_rows: L > 1024 not built");
    cudaError_t e = launch_softmax_rows(S, ldS, strideS, static_cast<__nv_bfloat16 *>(P), ldP, strideP, batch, rows, L,
                                        static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_softmax_rows launch", e);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_layernorm(const void *X, int64_t ldx, const float *gamma, const float *beta, float eps, void *Y,
                                int64_t ldy, int64_t rows, int64_t d, void *stream) {
    if (!X || !gamma || !beta || !Y) return fail(NIMBLE_E_NULL, "nimble_layernorm: NULL pointer");
    if (!ext_ok(rows) || !ext_ok(d)) return fail(NIMBLE_E_EXTENT, "nimble_layernorm: extents must be >= 1");
    if (d > 4096) return fail(NIMBLE_E_UNSUPPORTED, "nimble_layernorm: d > 4096 not built");
    if (d % 8 || ldx % 8 || ldy % 8 || !aligned16(X) || !aligned16(Y) || !aligned16(gamma) || !aligned16(beta))
        return fail(NIMBLE_E_ALIGN, "nimble_layernorm: d, ldx, ldy multiples of 8; X, Y, gamma, beta 16-B aligned");
    cudaError_t e = launch_layernorm(static_cast<const __nv_bfloat16 *>(X), ldx, gamma, beta, eps,
                                     static_cast<__nv_bfloat16 *>(Y), ldy, rows, d, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_layernorm launch", e);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_layernorm_dev(const void *X, int64_t ldx, const float *gamma, const float *beta, float eps,
                                    void *Y, int64_t ldy, const int32_t *rows_dev, int64_t rows_max, int64_t d,
                                    void *stream) {
    if (!X || !gamma || !beta || !Y || !rows_dev) return fail(NIMBLE_E_NULL, "nimble_layernorm_dev: NULL pointer");
    if (!ext_ok(rows_max) || !ext_ok(d)) return fail(NIMBLE_E_EXTENT, "nimble_layernorm_dev: extents must be >= 1");
    if (d > 4096) return fail(NIMBLE_E_UNSUPPORTED, "nimble_layernorm_dev: d > 4096 not built");
    if (d % 8 || ldx % 8 || ldy % 8 || !aligned16(X) || !aligned16(Y) || !aligned16(gamma) || !aligned16(beta))
        return fail(NIMBLE_E_ALIGN, "nimble_layernorm_dev: d, ldx, ldy multiples of 8; X, Y, gamma, beta 16-B aligned");
    cudaError_t e = launch_layernorm(static_cast<const __nv_bfloat16 *>(X), ldx, gamma, beta, eps,
                                     static_cast<__nv_bfloat16 *>(Y), ldy, rows_max, d,
                                     static_cast<cudaStream_t>(stream), rows_dev);
    if (e != cudaSuccess) return cuda_fail("nimble_layernorm_dev launch", e);
    clear_error();
    return NIMBLE_OK;
}

// ------------------------------------------------------------------ LSTM
extern "C" size_t nimble_lstm_workspace_bytes(int64_t H) { return H >= 1 ? lstm_workspace_bytes(H) : 0; }

extern "C" int nimble_lstm_seq(const float *G, int64_t ldg, const float *W_hh, int64_t ldw, const float *h0,
                               const float *c0, float *H_seq, int64_t ldh, float *hT, float *cT, int64_t T, int64_t H,
                               void *workspace, void *stream) {
    if (!G || !W_hh || !H_seq || !hT || !cT || !workspace) return fail(NIMBLE_E_NULL, "nimble_lstm_seq: NULL pointer");
    if (!ext_ok(T) || !ext_ok(H)) return fail(NIMBLE_E_EXTENT, "nimble_lstm_seq: T and H must be >= 1");
    if (ldg < 4 * H || ldw < H || ldh < H) return fail(NIMBLE_E_SHAPE, "nimble_lstm_seq: leading dimension too small");
    if (H > 4096) return fail(NIMBLE_E_UNSUPPORTED, "nimble_lstm_seq: H > 4096 not built");
    cudaError_t e = launch_lstm_seq(G, ldg, W_hh, ldw, h0, c0, H_seq, ldh, hT, cT, T, H, workspace,
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_lstm_seq launch", e);
    clear_error();
    return NIMBLE_OK;
}

extern "C" size_t nimble_lstm2_workspace_bytes(int64_t H) { return H >= 1 ? lstm2_workspace_bytes(H) : 0; }

extern "C" int nimble_lstm2_seq(const float *G1, int64_t ldg, const float *W_hh1, const float *W_ih2,
                                const float *W_hh2, int64_t ldw, const float *b2, float *H1, float *H2, int64_t ldh,
                                float *hT, float *cT, int64_t T, int64_t H, void *workspace, void *stream) {
    if (!G1 || !W_hh1 || !W_ih2 || !W_hh2 || !b2 || !H1 || !H2 || !hT || !cT || !workspace)
        return fail(NIMBLE_E_NULL, "nimble_lstm2_seq: NULL pointer");
    if (!ext_ok(T) || !ext_ok(H)) return fail(NIMBLE_E_EXTENT, "nimble_lstm2_seq: T and H must be >= 1");
    if (ldg < 4 * H || ldw < H || ldh < H) return fail(NIMBLE_E_SHAPE, "nimble_lstm2_seq: leading dimension too small");
    if (H > 1024) return fail(NIMBLE_E_UNSUPPORTED, "nimble_lstm2_seq: H > 1024 not built");
    cudaError_t e = launch_lstm2_seq(G1, ldg, W_hh1, W_ih2, W_hh2, ldw, b2, H1, H2, ldh, hT, cT, T, H, workspace,
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_lstm2_seq launch", e);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_lstm2_forward(const float *X, int64_t ldx, int64_t I, const float *W_ih1, int64_t ldwi,
                                    const float *b1, const float *W_hh1, const float *W_ih2, const float *W_hh2,
                                    int64_t ldw, const float *b2, float *H1, float *H2, int64_t ldh, float *hT,
                                    float *cT, int64_t T, int64_t H, void *workspace, void *stream) {
    if (!X || !W_ih1 || !b1 || !W_hh1 || !W_ih2 || !W_hh2 || !b2 || !H1 || !H2 || !hT || !cT || !workspace)
        return fail(NIMBLE_E_NULL, "nimble_lstm2_forward: NULL pointer");
    if (!ext_ok(T) || !ext_ok(H) || !ext_ok(I)) return fail(NIMBLE_E_EXTENT, "nimble_lstm2_forward: T, H and I must be >= 1");
    if (ldx < I || ldwi < I || ldw < H || ldh < H) return fail(NIMBLE_E_SHAPE, "nimble_lstm2_forward: leading dimension too small");
    const Lstm2Input in{X, ldx, W_ih1, ldwi, b1, I};
    cudaError_t e = launch_lstm2_seq(nullptr, 0, W_hh1, W_ih2, W_hh2, ldw, b2, H1, H2, ldh, hT, cT, T, H, workspace,
                                     static_cast<cudaStream_t>(stream), &in);
    if (e == cudaErrorNotSupported)
        return fail(NIMBLE_E_UNSUPPORTED, "nimble_lstm2_forward: H <= 672 and W_ih1 rows in shared memory required "
                                          "(use nimble_dense_dyn + nimble_lstm2_seq)");
    if (e != cudaSuccess) return cuda_fail("nimble_lstm2_forward launch", e);
    clear_error();
    return NIMBLE_OK;
}

// ------------------------------------------------------------------ Tree-LSTM
extern "C" int nimble_treelstm_level(const int32_t *nodes, const float *A, int64_t lda, const int32_t *a_rows,
                                     const float *W, int64_t ldw, const float *bias, const int32_t *parent_slot,
                                     float *hcat, float *ccat, int64_t ldcat, float *h_out, float *c_out, int64_t ldo,
                                     int64_t M, int64_t K, int64_t H, int is_leaf, void *stream) {
    if (!nodes || !A || !a_rows || !W || !bias || !parent_slot || !hcat || !ccat || !h_out || !c_out)
        return fail(NIMBLE_E_NULL, "nimble_treelstm_level: NULL pointer");
    if (!ext_ok(M) || !ext_ok(K) || !ext_ok(H)) return fail(NIMBLE_E_EXTENT, "nimble_treelstm_level: extents must be >= 1");
    if (!is_leaf && K != 2 * H) return fail(NIMBLE_E_SHAPE, "nimble_treelstm_level: internal nodes need K == 2H");
    if (lda < K || ldw < K || ldcat < 2 * H || ldo < H) return fail(NIMBLE_E_SHAPE, "nimble_treelstm_level: ld too small");
    if (!aligned16(A) || !aligned16(W) || lda % 4 || ldw % 4 || K % 4)
        return fail(NIMBLE_E_ALIGN, "nimble_treelstm_level: A/W need 16-B alignment, lda, ldw, K multiples of 4");
    TreeParams p{nodes, A, lda, a_rows, W, ldw, bias, parent_slot, hcat, ccat, ldcat, h_out, c_out, ldo,
                 (int32_t)M, (int32_t)K, (int32_t)H, is_leaf};
    cudaError_t e = launch_treelstm_level(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_treelstm_level launch", e);
    clear_error();
    return NIMBLE_OK;
}

extern "C" int nimble_treelstm_forest(const float *X, int64_t ldx, const float *W_l, const float *b_l, const float *U,
                                      const float *b_u, int64_t I, int64_t H, const int32_t *level_off,
                                      int64_t n_levels, int64_t max_level, const int32_t *nodes, const int32_t *rows,
                                      const int32_t *parent_slot, float *hcat, float *ccat, int64_t ldcat,
                                      float *h_out, float *c_out, int64_t ldo, void *workspace, void *stream) {
    if (!X || !W_l || !b_l || !U || !b_u || !level_off || !nodes || !rows || !parent_slot || !hcat || !ccat ||
        !h_out || !c_out || !workspace)
        return fail(NIMBLE_E_NULL, "nimble_treelstm_forest: NULL pointer");
    if (!ext_ok(I) || !ext_ok(H) || !ext_ok(n_levels) || !ext_ok(max_level))
        return fail(NIMBLE_E_EXTENT, "nimble_treelstm_forest: extents must be >= 1");
    if (ldx < I || ldcat < 2 * H || ldo < H) return fail(NIMBLE_E_SHAPE, "nimble_treelstm_forest: ld too small");
    if (!aligned16(X) || !aligned16(W_l) || !aligned16(U) || !aligned16(hcat) || ldx % 4 || ldcat % 4 || I % 4 ||
        (2 * H) % 4)
        return fail(NIMBLE_E_ALIGN, "nimble_treelstm_forest: X/W_l/U/hcat need 16-B alignment; ldx, ldcat, I, 2H multiples of 4");
    TreeForestParams p{X, ldx, W_l, b_l, U, b_u, level_off, nodes, rows, parent_slot, hcat, ccat, ldcat, h_out, c_out,
                       ldo, static_cast<unsigned *>(workspace), nullptr, (int32_t)n_levels, (int32_t)I, (int32_t)H,
                       (int32_t)max_level};
    cudaError_t e = launch_treelstm_forest(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("nimble_treelstm_forest launch", e);
    clear_error();
    return NIMBLE_OK;
}
