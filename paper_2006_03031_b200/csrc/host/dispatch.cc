// The generated dispatch function of Nimble §3.5: the symbolic
// extent x is split as x = t*k + r and the residue picks a specialised kernel;
// with a variant limit c < n_classes "fewer kernels than the tiling factor" exist
// (fig:sym-codegen PAPER.md:699) and the rest take the guarded
// fallback.  The rule is DISPATCH.md; the oracle implements it independently.
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.h"

namespace nimble {

static std::atomic<int> g_variant_limit{0};

int variant_limit() { return g_variant_limit.load(std::memory_order_relaxed); }

namespace {

struct ResidueFamily {
    int32_t id, t, granule, n_classes;
};
constexpr ResidueFamily kSIMT8{0, 8, 1, 8};      // fp32 CUDA-core dense, the paper's t = 8
constexpr ResidueFamily kUMMA_T{1, 128, 16, 9};    // bf16 tcgen05, tokens on UMMA-N (128 x 128 tiles)
constexpr ResidueFamily kUMMA_T256{3, 256, 16, 17}; // same, CTA pairs (256 x 256 tiles, no split-K)
constexpr int64_t kScheduleBelow = 2048;            // tuned family-1 schedules cover M < 2048
constexpr ResidueFamily kUMMA_D{2, 128, 128, 2}; // bf16 tcgen05 bmm with MN-major B
constexpr ResidueFamily kUMMA_WS{4, 128, 16, 9};  // bf16 tcgen05 dense, M <= 128: weight streaming

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// class -> specialised variant, or -1 when the variant limit leaves it to the fallback
int32_t select_variant(const ResidueFamily &f, int32_t cls) {
    const int c = variant_limit();
    const int kernels = (c <= 0 || c > f.n_classes) ? f.n_classes : c;
    const bool specialised = (kernels == f.n_classes) || (cls <= kernels - 2);
    return specialised ? cls : -1;
}

// split-K factor (cluster size along K): grow while the grown grid still fits one
// wave of 148 CTAs and every split keeps >= 4 k-blocks of 64; at most `cap`.
int32_t choose_split(int64_t ctas, int64_t K, int32_t cap = 8) {
    const int64_t kblocks = cdiv(K, 64);
    int32_t s = 1;
    for (;;) {
        const int32_t next = s * 2;
        if (next > cap || ctas * next > kNumSMs || kblocks / next < 4) break;
        s = next;
    }
    return s;
}

// The default split cap: split-K only for K >= 2048.  Below that the DSMEM exchange of the
// fp32 partial tiles costs more than the shorter K loop saves at M >= 64 (measured on B200:
// profiles/r01_gemm_sweep.json, P:392-406 tuning data in profiles/r01_symbolic_tuning.json;
// at M <= 16 the split would still win — the tuned schedules cover that).  A cap depending on
// K alone keeps the split a function of the tile grid, so dynamic M stays bit-identical to
// pad-then-slice.  Tuned schedules carry their own cap.
int32_t default_split_cap(int64_t M, int64_t K) { (void)M; return K >= 2048 ? 8 : 1; }

void split_residue(const ResidueFamily &f, int64_t x, nimble_dispatch *d) {
    d->family = f.id;
    d->tile_t = f.t;
    d->granule = f.granule;
    d->n_classes = f.n_classes;
    d->k = x / f.t;                 // x = t*k + r
    d->r = x - d->k * f.t;
}

}  // namespace

int dispatch_simt8(int64_t M, int64_t N, nimble_dispatch *d) {
    *d = nimble_dispatch{};
    split_residue(kSIMT8, M, d);
    d->residue_class = static_cast<int32_t>(d->r);
    d->variant = select_variant(kSIMT8, d->residue_class);
    d->split_k = 1;
    d->grid[0] = static_cast<int32_t>(cdiv(N, 32));     // 32 output features per CTA (4 warps split K)
    d->grid[1] = static_cast<int32_t>(d->k + (d->r ? 1 : 0));
    d->grid[2] = 1;
    d->cluster[0] = d->cluster[1] = d->cluster[2] = 1;
    return NIMBLE_OK;
}

// Family 3 iff its 256 x 256 pair tiles need fewer waves (74 CTA pairs) than family 1's
// 128 x 128 tiles (148 CTAs): measured on B200 (profiles/r02e_f1_vs_f3.jsonl), a pair tile at
// K >= 768 costs about what a family-1 tile costs (both paced by the per-stage TMA feed,
// DESIGN.md §6), so the family with fewer waves wins at every BERT shape for M = 768-8192; with
// equal waves family 1 is faster (half the work per CTA).  Replaces the round-1 threshold M >= 2048.
bool pair_rule(int64_t batch, int64_t M, int64_t N) {
    const int64_t t1 = cdiv(N, 128) * cdiv(M, 128) * batch;
    const int64_t t3 = cdiv(N, 256) * cdiv(M, 256) * batch;
    return cdiv(t3, kNumSMs / 2) < cdiv(t1, kNumSMs);
}

int dispatch_umma_t(int64_t batch, int64_t M_tokens, int64_t N_rows, int64_t K, nimble_dispatch *d,
                    int32_t tile_t, int32_t split_max) {
    *d = nimble_dispatch{};
    // family 3 (CTA pairs, 256 x 256 tiles) where it needs fewer waves than family 1's 128 x 128
    // tiles (pair_rule); a tuned schedule replaces the default rule below M = 2048
    const bool sched = tile_t > 0 && M_tokens < kScheduleBelow;
    bool wide = !sched && pair_rule(batch, M_tokens, N_rows);
    // experiment-only overrides (break oracle parity): NIMBLE_EXP_PAIR_FROM replaces the rule by
    // a token threshold, NIMBLE_EXP_T3 sets family 3's token tile
    static const int64_t pair_from = [] { const char *e = std::getenv("NIMBLE_EXP_PAIR_FROM"); return e ? std::atoll(e) : 0; }();
    static const int32_t t3 = [] { const char *e = std::getenv("NIMBLE_EXP_T3"); return e ? std::atoi(e) : kUMMA_T256.t; }();
    if (pair_from > 0) wide = M_tokens >= pair_from;
    const ResidueFamily tuned{kUMMA_T.id, tile_t, 16, tile_t / 16 + 1};
    const ResidueFamily wide_f{kUMMA_T256.id, t3, 16, t3 / 16 + 1};
    const ResidueFamily &f = wide ? wide_f : (sched ? tuned : kUMMA_T);
    // split-K parks and receives fp32 [128 x t] slices in smem: only t <= 128 fits 227 KB
    const int32_t cap = sched ? (tile_t <= 128 ? split_max : 1) : default_split_cap(M_tokens, K);
    split_residue(f, M_tokens, d);
    d->residue_class = static_cast<int32_t>(cdiv(d->r, f.granule));
    d->variant = select_variant(f, d->residue_class);
    d->umma_m = 128;
    d->umma_n_full = f.t;
    d->umma_n_tail = d->r == 0 ? 0 : (d->variant < 0 ? f.t : f.granule * d->residue_class);
    const int64_t m_tiles = cdiv(N_rows, 128);
    const int64_t n_tiles = d->k + (d->r ? 1 : 0);
    d->split_k = (f.id == kUMMA_T.id) ? choose_split(m_tiles * n_tiles * batch, K, cap) : 1;
    static const int force = [] { const char *e = std::getenv("NIMBLE_FORCE_SPLIT"); return e ? std::atoi(e) : 0; }();
    if (force > 0) d->split_k = force;      // experiment-only override (breaks oracle parity)
    d->grid[0] = static_cast<int32_t>(m_tiles);
    d->grid[1] = static_cast<int32_t>(n_tiles);
    d->grid[2] = static_cast<int32_t>(batch * d->split_k);
    const bool pair = (f.id == kUMMA_T256.id);             // family 3: CTA pairs, cta_group::2
    d->umma_m = pair ? 256 : 128;
    d->cluster[0] = pair ? 2 : 1;
    d->cluster[1] = 1;
    d->cluster[2] = d->split_k;
    return NIMBLE_OK;
}

// Family 4 (DISPATCH.md): a dense without a tuned schedule whose (feature tile, token tile)
// units leave most SMs idle streams its weights over one wave of CTAs: units x S splits of K
// (one cluster per unit, S <= 8), S a function of (N, K, ceil(M / 128)) only.
#ifndef NIMBLE_WS_MAX_CLUSTER
#define NIMBLE_WS_MAX_CLUSTER 8
#endif
// the largest PORTABLE thread-block cluster: 16-CTA (non-portable) clusters measured up to 20 %
// faster on the K >= 3072 shapes but 8 clusters of 16 fill all 8 GPCs exactly, and
// compute-sanitizer synccheck flags them ("missing wait"); 8-CTA clusters are clean
constexpr int64_t kWsMaxCluster = NIMBLE_WS_MAX_CLUSTER;
constexpr int64_t kWsMaxTokenTiles = 8;          // M <= 1024

int64_t ws_split(int64_t units, int64_t K) {
    int64_t s = kNumSMs / units;                    // one wave of CTAs ...
    const int64_t kb = cdiv(K, 64);
    if (s > kb) s = kb;                             // ... each with >= 1 k-block of 64 ...
    if (s > kWsMaxCluster) s = kWsMaxCluster;       // ... the splits of a unit one cluster
    return s < 1 ? 1 : s;
}

// one token tile: whenever the feature tiles fit one wave; 2..8 token tiles: where family 1
// would split K (K >= 2048) and the split stays >= 2 (fewer than 75 units).  Measured on B200
// (profiles/r02_ws_sweep.jsonl): at K <= 1024 the 128-token partial exchange costs more than
// family 1's whole K loop; at K >= 2048 the L2 + cluster-barrier exchange beats family 1's
// DSMEM split-K by 1.2-2.3x.
bool ws_applies(int64_t M, int64_t N, int64_t K) {
    const int64_t n_tiles = cdiv(M, kUMMA_WS.t), m_tiles = cdiv(N, 128);
    if (n_tiles == 1) return m_tiles <= kNumSMs;
    return n_tiles <= kWsMaxTokenTiles && K >= 2048 && ws_split(m_tiles * n_tiles, K) >= 2;
}

int dispatch_umma_ws(int64_t M, int64_t N, int64_t K, nimble_dispatch *d) {
    *d = nimble_dispatch{};
    split_residue(kUMMA_WS, M, d);
    d->residue_class = static_cast<int32_t>(cdiv(d->r, kUMMA_WS.granule));
    d->variant = select_variant(kUMMA_WS, d->residue_class);
    d->umma_m = 128;
    d->umma_n_full = kUMMA_WS.t;
    d->umma_n_tail = d->r == 0 ? 0 : (d->variant < 0 ? kUMMA_WS.t : kUMMA_WS.granule * d->residue_class);
    const int64_t m_tiles = cdiv(N, 128);
    const int64_t n_tiles = d->k + (d->r ? 1 : 0);
    d->split_k = static_cast<int32_t>(ws_split(m_tiles * n_tiles, K));
    d->grid[0] = static_cast<int32_t>(m_tiles);
    d->grid[1] = static_cast<int32_t>(n_tiles);
    d->grid[2] = d->split_k;
    d->cluster[0] = d->cluster[1] = d->cluster[2] = 1;
    return NIMBLE_OK;
}

int dispatch_dense_bf16(int64_t M, int64_t N, int64_t K, nimble_dispatch *d) {
    int32_t t, cap;
    dense_schedule(N, K, &t, &cap);
    if (t == 0 && ws_applies(M, N, K)) return dispatch_umma_ws(M, N, K, d);
    return dispatch_umma_t(1, M, N, K, d, t, cap);
}

int dispatch_umma_d(int64_t batch, int64_t M, int64_t N, int64_t K, nimble_dispatch *d) {
    *d = nimble_dispatch{};
    split_residue(kUMMA_D, M, d);
    d->residue_class = d->r ? 1 : 0;
    d->variant = select_variant(kUMMA_D, d->residue_class);
    d->umma_m = 128;
    const int64_t n_tiles = cdiv(N, 256);
    d->umma_n_full = static_cast<int32_t>(N >= 256 ? 256 : 16 * cdiv(N, 16));
    d->umma_n_tail = static_cast<int32_t>(16 * cdiv(N - 256 * (n_tiles - 1), 16));
    const int64_t m_tiles = d->k + (d->r ? 1 : 0);
    d->split_k = choose_split(m_tiles * n_tiles * batch, K, default_split_cap(M, K));
    d->grid[0] = static_cast<int32_t>(m_tiles);
    d->grid[1] = static_cast<int32_t>(n_tiles);
    d->grid[2] = static_cast<int32_t>(batch * d->split_k);
    d->cluster[0] = 1;
    d->cluster[1] = 1;
    d->cluster[2] = d->split_k;
    return NIMBLE_OK;
}

// ---------------------------------------------------------------- tuned schedules
namespace {
struct ScheduleEntry {
    int64_t N, K;
    int32_t tile_t, split_max;
};
std::mutex g_sched_mu;
std::vector<ScheduleEntry> g_sched;
}  // namespace

void dense_schedule(int64_t N, int64_t K, int32_t *tile_t, int32_t *split_max) {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    *tile_t = 0;
    *split_max = 8;
    for (const auto &e : g_sched)
        if (e.N == N && e.K == K) {
            *tile_t = e.tile_t;
            *split_max = e.split_max;
            return;
        }
}

}  // namespace nimble

using namespace nimble;

extern "C" int nimble_set_dense_schedule(int64_t N, int64_t K, int32_t tile_t, int32_t split_max) {
    if (N < 1 || K < 1 || N > kMaxExtent || K > kMaxExtent)
        return fail(NIMBLE_E_EXTENT, "nimble_set_dense_schedule: extents must be in [1, 2^31-1]");
    if (tile_t != 0 && tile_t != 32 && tile_t != 64 && tile_t != 128 && tile_t != 256)
        return fail(NIMBLE_E_EXTENT, "nimble_set_dense_schedule: tile_t must be 0, 32, 64, 128 or 256");
    if (split_max != 1 && split_max != 2 && split_max != 4 && split_max != 8)
        return fail(NIMBLE_E_EXTENT, "nimble_set_dense_schedule: split_max must be 1, 2, 4 or 8");
    std::lock_guard<std::mutex> lk(g_sched_mu);
    for (size_t i = 0; i < g_sched.size(); ++i)
        if (g_sched[i].N == N && g_sched[i].K == K) {
            if (tile_t == 0) g_sched.erase(g_sched.begin() + (long)i);
            else g_sched[i].tile_t = tile_t, g_sched[i].split_max = split_max;
            return NIMBLE_OK;
        }
    if (tile_t != 0) g_sched.push_back({N, K, tile_t, split_max});
    return NIMBLE_OK;
}

extern "C" int nimble_get_dense_schedule(int64_t N, int64_t K, int32_t *tile_t, int32_t *split_max) {
    if (!tile_t || !split_max) return fail(NIMBLE_E_NULL, "nimble_get_dense_schedule: NULL output");
    dense_schedule(N, K, tile_t, split_max);
    return NIMBLE_OK;
}

static bool extents_valid(std::initializer_list<int64_t> xs) {
    for (int64_t x : xs)
        if (x < 1 || x > kMaxExtent) return false;
    return true;
}

extern "C" int nimble_set_variant_limit(int c) {
    if (c < 0) return fail(NIMBLE_E_EXTENT, "nimble_set_variant_limit: c must be >= 0");
    g_variant_limit.store(c);
    return NIMBLE_OK;
}

extern "C" int nimble_get_variant_limit(void) { return variant_limit(); }

extern "C" int nimble_dispatch_dense(int64_t M, int64_t N, int64_t K, int dt, nimble_dispatch *out) {
    if (!out) return fail(NIMBLE_E_NULL, "nimble_dispatch_dense: out is NULL");
    if (!extents_valid({M, N, K})) return fail(NIMBLE_E_EXTENT, "nimble_dispatch_dense: extents must be in [1, 2^31-1]");
    if (dt == NIMBLE_F32) return dispatch_simt8(M, N, out);
    if (dt == NIMBLE_BF16) return dispatch_dense_bf16(M, N, K, out);
    return fail(NIMBLE_E_DTYPE, "nimble_dispatch_dense: unknown dtype");
}

extern "C" int nimble_dispatch_bmm(int64_t batch, int64_t M, int64_t N, int64_t K, int trans_b, int dt,
                                   nimble_dispatch *out) {
    if (!out) return fail(NIMBLE_E_NULL, "nimble_dispatch_bmm: out is NULL");
    if (!extents_valid({batch, M, N, K})) return fail(NIMBLE_E_EXTENT, "nimble_dispatch_bmm: extents must be in [1, 2^31-1]");
    if (dt == NIMBLE_F32) return fail(NIMBLE_E_UNSUPPORTED, "nimble_dispatch_bmm: fp32 bmm is not built (bf16 only)");
    if (dt != NIMBLE_BF16) return fail(NIMBLE_E_DTYPE, "nimble_dispatch_bmm: unknown dtype");
    return trans_b ? dispatch_umma_d(batch, M, N, K, out) : dispatch_umma_t(batch, M, N, K, out);
}
