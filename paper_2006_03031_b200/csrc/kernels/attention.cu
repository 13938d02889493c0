// Fused variable-length attention over token-packed requests:
// for every request i (tokens [o_i, o_i + L_i) of a packed QKV [T x 3d]) and head h,
//     C_h = softmax(Q_h K_h^T * scale) V_h
// in ONE launch, with L_i a per-request symbolic extent (PAPER.md:255 one symbol for the
// equal dynamic dims; P:575 BERT's dynamic sequence length).  It replaces the
// bmm_dyn -> softmax_rows -> bmm_dyn triple and never writes S or P to HBM.
//
// Persistent: two CTAs per SM walk a shared list of work items (query tile of 128, head,
// request).  Every CTA builds the same list from seq_off in its prologue — requests ordered
// by key-block count, longest first (a stable counting sort), items of one (request, head)
// adjacent so concurrently running CTAs share K/V in L2 — and takes items
// blockIdx.x, blockIdx.x + gridDim.x, ...  The TMEM allocation, barrier setup and tensor-map
// prefetch happen once per CTA, and the producer runs ahead into the next item (its Q and
// first K/V blocks load while the current item finishes).
// Per item, online softmax over 128-key blocks, 320 threads:
//   warp 8 lane 0  TMA producer and the only role that decodes the work list: publishes each
//                  item's (offset, L, q-tile, head) in a 2-slot smem ring released by the Q
//                  barrier; Q tile, then per key block K_j [128 x 64] (single buffer) and V_j
//                  (MN-major, two 64-key boxes, 2-stage ring).
//   warp 9 lane 0  MMA issuer: S = Q K_j^T into TMEM cols [0,128) as soon as the previous S
//                  has been read (the next item's first S before this item's last PV);
//                  O += P_j V_j into TMEM cols [128,192) once P_j is written.
//   warps 0-7      softmax: row q = TMEM lane 32*(w%4)+lane, key half (w/4) of the block held
//                  in registers; running max / sum in FFMA2 / FADD2 / FMNMX3, exp2 on MUFU
//                  and (3 of 8 pairs) on the FMA pipes; unnormalised P_j written as bf16
//                  straight into the UMMA K-major swizzled smem layout; O rescaled in TMEM
//                  only when a row max grew by more than 2^8 (lazy rescaling); epilogue
//                  O / rowsum -> bf16.
// TMEM 256 columns and ~113 KB smem per CTA: two CTAs share an SM.  Keys >= L_i get P = 0;
// query rows >= L_i are computed but never stored.
#include <cstdint>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kSoftmaxThreads = 256;     // warps 0-7
// + warp 8 (lane 0: TMA producer) and warp 9 (lane 0: MMA issuer).  The two spin-waiting roles
// must not share a warp: divergent lanes of one warp are scheduled one path at a time, so a
// producer spinning on an mbarrier would delay the MMA issue (and vice versa) by microseconds.
constexpr int kThreads = kSoftmaxThreads + 64;
constexpr int kTile = 128 * 64 * 2;       // Q tile / K block / V block (128 keys) / P half: 16 KiB
constexpr int kVBox = 64 * 64 * 2;        // one V TMA box (64 keys): 8 KiB
constexpr int kMaxReq = 1024;             // requests per launch (work-list arrays in smem)
constexpr int kMaxQT = 64;                // query tiles per request (max_len <= 8192)
constexpr int kRedBytes = 4 * 256 * 4;    // [2 parity][2 halves][128] row max + [2][128] row sums
// rounded to 1 KiB: the barrier block after it holds the 128-B-aligned maps being patched
constexpr int kListBytes = (2 * kMaxReq * 4 + kMaxReq * 2 + 2 * (kMaxQT + 1) * 4 + 1023) / 1024 * 1024;
constexpr int kSmemBytes = 1024 + 6 * kTile + kRedBytes + kListBytes + 512;   // + barriers, 2 map scratches
constexpr int kCtasPerSm = 2;
constexpr uint32_t kPCol = 192;           // TMEM column of P_j (128 x 128 bf16 = 64 columns)

// TMA maps of the output with boxes of 64, 32, 16 and 8 rows: a partial query tile's valid
// rows leave as a 64/32/16/8-row decomposition (starting rows stay multiples of 8, so every
// box starts on a 1 KB swizzle atom of the staging); only the last < 8 rows use plain stores.
struct OutMaps {
    CUtensorMap box[4];
};

struct AttnParams {
    const int32_t *seq_off;   // [R + 1] prefix sums of request lengths (device)
    int32_t R;
    int32_t heads;
    float scale_log2;         // scale * log2(e)
    __nv_bfloat16 *out;
    int64_t ld_out;
    CUtensorMap *map_slots;   // patch_T: 2 per-CTA slots for the extent-patched Q/K and V maps
    int32_t patch_T;          // device token count: re-encode the Q/K and V maps with T = seq_off[R]
    int32_t T_max;            // bound on seq_off[R] (the tensor maps' / output's row extent)
    int32_t max_len;          // bound on every L_i
    unsigned long long *trace;   // debug (nimble_debug_trace): CTA 0 per-block clock64 stamps
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 32 lanes x 32 consecutive columns (lane i of the warp -> TMEM lane base + i)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: A is a 128 x 16 bf16 tile in TMEM (lane = row, two k per
// 32-bit column: 8 columns), B the usual shared-memory descriptor
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

using ptx::fadd2;
using ptx::ffma2;
using ptx::fmax3;

// 2^x for x <= 0 on the FMA pipes (a pair at a time): x = j + f, j = rint(x) by the 1.5 * 2^23
// magic-number rounding, f in [-1/2, 1/2]; 2^f by a degree-3 minimax polynomial (relative
// error 7.5e-5, far below the bf16 rounding of P); 2^j added into the exponent field.  x is
// clamped at -125 so the exponent stays normal (2^-125 is 0 next to a row sum >= 1).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 magic = make_float2(12582912.f, 12582912.f), nmagic = make_float2(-12582912.f, -12582912.f);
    const float2 t = fadd2(x, magic);
    const float2 r = fadd2(t, nmagic);                           // rint(x)
    const float2 f = fadd2(x, make_float2(-r.x, -r.y));
    float2 q = ffma2(make_float2(0.0551710878f, 0.0551710878f), f, make_float2(0.242611162f, 0.242611162f));
    q = ffma2(q, f, make_float2(0.693261098f, 0.693261098f));
    q = ffma2(q, f, make_float2(0.999928072f, 0.999928072f));
    return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
#ifndef NIMBLE_ATTN_LAZY
#define NIMBLE_ATTN_LAZY 8.0f        // lazy-rescale threshold (log2 units); 0 = rescale on every growth
#endif
constexpr float kLazy = NIMBLE_ATTN_LAZY;
#ifndef NIMBLE_ATTN_POLY
#define NIMBLE_ATTN_POLY 3          // pairs out of every 8 whose exp2 runs on the FMA pipes (3: 65.3 vs 65.6 us, r02e_attn_poly_ab.txt)
#endif

__device__ __forceinline__ int qtiles_of(const int32_t *seq_off, int r) {
    const int L = __ldg(seq_off + r + 1) - __ldg(seq_off + r);
    return (L + 127) / 128;
}

// The work list: requests ordered by query-tile count, descending (stable); per sorted position
// i: so[i] = token offset, sl[i] = length, cum[i] = items of positions [0, i).  Item k -> the i
// with cum[i] <= k < cum[i+1]; within a request, q-tile fastest.  Decoding touches shared memory
// only: a dependent global load at an item boundary stalls every role for microseconds.
struct Item {
    int o, L, qt, h;
};
__device__ __forceinline__ Item decode_item(const int32_t *so, const int16_t *sl, const int32_t *cum, int R, int heads,
                                            int k) {
    int lo = 0, hi = R - 1;                        // largest i with cum[i] <= k
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cum[mid] <= k) lo = mid;
        else hi = mid - 1;
    }
    Item it;
    it.o = so[lo];
    it.L = sl[lo];
    const int nq = (it.L + 127) / 128;
    const int rem = k - cum[lo];
    it.qt = rem % nq;
    it.h = rem / nq;
    return it;
}

// This CTA's items k = blockIdx.x + n * gridDim.x.  Decoding is kept off the item boundary:
// lookahead() decodes the item after next somewhere inside the current item (where the role
// would be waiting anyway) and advance() only moves registers.  Shared-memory loads of the
// single-thread roles queue behind the softmax warps' MUFU traffic in the MIO pipe, so a
// decode at the boundary costs thousands of cycles.
struct ItemIter {
    const int32_t *so, *cum;
    const int16_t *sl;
    int R, H, n, k;
    Item cur, nxt, nxt2;
    __device__ __forceinline__ ItemIter(const int32_t *so_, const int16_t *sl_, const int32_t *cum_, int R_, int H_,
                                        int n_)
        : so(so_), cum(cum_), sl(sl_), R(R_), H(H_), n(n_), k((int)blockIdx.x) {
        if (k < n) cur = decode_item(so, sl, cum, R, H, k);
        if (k + (int)gridDim.x < n) nxt = decode_item(so, sl, cum, R, H, k + (int)gridDim.x);
    }
    __device__ __forceinline__ bool valid() const { return k < n; }
    __device__ __forceinline__ bool has_next() const { return k + (int)gridDim.x < n; }
    __device__ __forceinline__ void lookahead() {
        if (k + 2 * (int)gridDim.x < n) nxt2 = decode_item(so, sl, cum, R, H, k + 2 * (int)gridDim.x);
    }
    __device__ __forceinline__ void advance() {
        k += (int)gridDim.x;
        cur = nxt;
        nxt = nxt2;
    }
};

__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    attention_varlen_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                            const __grid_constant__ CUtensorMap tmO, const __grid_constant__ OutMaps tmOp,
                            const AttnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sQ = smem;
    uint8_t *sK = smem + kTile;                   // K block (single buffer: only the short S MMA reads it)
    uint8_t *sV = smem + 2 * kTile;               // [2] V blocks (two 64-key boxes each)
    uint8_t *sP = smem + 4 * kTile;               // P block: 2 x (64 keys) K-major atoms = 32 KiB
    float *red = reinterpret_cast<float *>(smem + 6 * kTile);           // [2 parity][2 halves][128] row max
    float *redl = red + 512;                                             // [2 halves][128] row sums
    int32_t *so = reinterpret_cast<int32_t *>(smem + 6 * kTile + kRedBytes);   // [R] sorted token offsets
    int32_t *cum = so + kMaxReq;                                         // [R + 1]
    int32_t *cnt = cum + kMaxReq;                                        // [kMaxQT + 1]
    int32_t *start = cnt + kMaxQT + 1;                                   // [kMaxQT + 1]
    int16_t *sl = reinterpret_cast<int16_t *>(start + kMaxQT + 1);       // [R] sorted lengths
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 6 * kTile + kRedBytes + kListBytes);
    uint64_t *q_full = bar, *q_empty = bar + 1, *k_full = bar + 2, *k_empty = bar + 3, *v_full = bar + 4,
             *v_empty = bar + 6, *s_full = bar + 8, *s_used = bar + 9, *p_ready = bar + 10, *pv_done = bar + 11,
             *o_free = bar + 12, *info_read = bar + 15;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 13);
    int4 *info = reinterpret_cast<int4 *>(bar + 16);                     // [2] published items (o, L, qt, h)
    uint8_t *smaps = reinterpret_cast<uint8_t *>(bar) + 256;            // 2 x 128-B maps being patched
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int R = p.R, H = p.heads;
    unsigned long long *trace = (p.trace && blockIdx.x == 0) ? p.trace : nullptr;
    const unsigned long long t_start = p.trace ? ptx::globaltimer() : 0ull;   // per-CTA span (debug)
    // debug timeline of CTA 0 (nimble_debug_trace): clock64 stamps kept in shared memory (the upper
    // half of the P buffer; the O staging uses the lower 16 KB) and copied out at the end, so the
    // trace adds no global stores (and no release-arrive waiting for them) on the hot path.
    // Slots: blocks 0-63, producer 256+n, MMA items 384+i, softmax items 448+i (n, i < 64).
    unsigned long long *strace = reinterpret_cast<unsigned long long *>(sP + 16384);
    auto trace_slot = [](int blk) { return blk < 64 ? blk : blk < 256 ? -1 : blk < 320 ? blk - 192 : blk < 384 ? -1
                                         : blk < 448 ? blk - 256 : blk < 512 ? blk - 256 : -1; };
#define ATT_TRACE(blk, ev) do { if (trace) { const int sl_ = trace_slot(blk); if (sl_ >= 0) strace[sl_ * 8 + (ev)] = clock64(); } } while (0)

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmQK);
        ptx::prefetch_tmap(&tmV);
        ptx::mbar_init(q_full, 1);
        ptx::mbar_init(q_empty, 1);
        ptx::mbar_init(k_full, 1);
        ptx::mbar_init(k_empty, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
        }
        ptx::mbar_init(s_full, 1);
        ptx::mbar_init(s_used, kSoftmaxThreads / 32);
        ptx::mbar_init(p_ready, kSoftmaxThreads / 32);
        ptx::mbar_init(pv_done, 1);
        ptx::mbar_init(o_free, kSoftmaxThreads / 32);
        ptx::mbar_init(info_read, kSoftmaxThreads / 32);
        ptx::fence_mbar_init();
        ptx::fence_async_smem();
    }
    if (warp == 8) ptx::tmem_alloc(tmem_slot, 256);
    if (trace)
        for (int i = threadIdx.x; i < 256 * 8; i += kThreads) strace[i] = 0ull;
    for (int i = threadIdx.x; i <= kMaxQT; i += kThreads) cnt[i] = 0;
    ptx::pdl_wait();                              // QKV and seq_off come from earlier work
    ptx::pdl_trigger();
    __syncthreads();
    // ---- seq_off is device data: a non-monotone prefix, an L_i above max_len or a total above
    //      the row extent the maps were encoded for would send TMA / row stores out of bounds
    for (int r = threadIdx.x; r < R; r += kThreads) {
        const int a = __ldg(p.seq_off + r), b = __ldg(p.seq_off + r + 1);
        if (a < 0 || b < a || b - a > p.max_len || b > p.T_max) __trap();
    }
    // ---- work list (identical in every CTA): counting sort of the requests by query tiles, descending
    for (int r = threadIdx.x; r < R; r += kThreads) atomicAdd(&cnt[min(qtiles_of(p.seq_off, r), kMaxQT)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int v = kMaxQT; v >= 0; --v) {
            start[v] = s;
            s += cnt[v];
        }
    }
    __syncthreads();
    if (warp == 0) {
        for (int base = 0; base < R; base += 32) {     // stable: requests placed in index order
            const int r = base + (int)lane;
            const int v = r < R ? min(qtiles_of(p.seq_off, r), kMaxQT) : -1;
            const uint32_t peers = __match_any_sync(0xffffffffu, v);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            if (r < R) {
                const int o = __ldg(p.seq_off + r);
                so[start[v] + rank] = o;
                sl[start[v] + rank] = (int16_t)(__ldg(p.seq_off + r + 1) - o);
            }
            __syncwarp();
            if (v >= 0 && (int)lane == __ffs(peers) - 1) start[v] += __popc(peers);
            __syncwarp();
        }
        int run = 0;                                    // cum: exclusive prefix of items per request
        for (int base = 0; base < R; base += 32) {
            const int i = base + (int)lane;
            int c = i < R ? ((int)sl[i] + 127) / 128 * H : 0;
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, d);
                if ((int)lane >= d) incl += t;
            }
            if (i < R) cum[i] = run + incl - c;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) cum[R] = run;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;             // S: cols [0,128), O: [128,192), P (bf16 pairs): [192,256)
    const int n_items = cum[R];

    // device token count (nimble_attention_varlen_dev): T = seq_off[R] is data, so this CTA
    // publishes copies of both maps with the token extent patched to T (rows past T then
    // zero-fill exactly as with a host-encoded T).
    const CUtensorMap *mQK = &tmQK, *mV = &tmV;
    if (p.patch_T && warp == 8) {
        const uint32_t T = (uint32_t)__ldg(p.seq_off + R);
        CUtensorMap *slot = p.map_slots + 2 * (size_t)blockIdx.x;
        mQK = ptx::tmap_patch_extent<2>(&tmQK, smaps, slot, T, lane);
        mV = ptx::tmap_patch_extent<2>(&tmV, smaps + 128, slot + 1, T, lane);
    }

    if (warp == 8) {
      if (lane == 0) {
        // ---------------- producer: the only role that decodes the work list.  Per item: publish
        // (o, L, qt, h) in info[n & 1], then Q once, then K_j / V_j; runs ahead into the next item.
        uint32_t nq = 0, nk_loaded = 0, nv = 0;
        for (ItemIter iter(so, sl, cum, R, H, n_items); iter.valid(); iter.advance()) {
            const Item it = iter.cur;
            const int nk = (it.L + 127) / 128;
            if (nq > 0) {
                ptx::mbar_wait(q_empty, (nq - 1) & 1);                      // last S of the previous item read Q
                // the softmax has read the previous item's info: q_full can never run two phases
                // ahead of a softmax waiter (its parity wait would then block on the wrong phase)
                ptx::mbar_wait(info_read, (nq - 1) & 1);
            }
            ATT_TRACE(256 + (int)nq, 0);
            info[nq & 1] = make_int4(it.o, it.L, it.qt, it.h);              // released by the q_full arrive
            ptx::mbar_arrive_expect_tx(q_full, kTile);
            ptx::tma_load_3d(sQ, mQK, q_full, 0, it.h, it.o + it.qt * 128);
            ++nq;
            for (int j = 0; j < nk; ++j) {
                if (nk_loaded > 0) ptx::mbar_wait(k_empty, (nk_loaded - 1) & 1);   // previous S read K
                ATT_TRACE(256 + (int)nk_loaded, 1);
                ptx::mbar_arrive_expect_tx(k_full, kTile);
                ptx::tma_load_3d(sK, mQK, k_full, 0, H + it.h, it.o + j * 128);
                ++nk_loaded;
                const int st = (int)(nv & 1), use = (int)(nv >> 1);
                if (use > 0) ptx::mbar_wait(&v_empty[st], (use - 1) & 1);   // PV two blocks back read V
                ATT_TRACE(256 + (int)nv, 2);
                ptx::mbar_arrive_expect_tx(&v_full[st], kTile);
                ptx::tma_load_3d(sV + st * kTile, mV, &v_full[st], 0, 2 * H + it.h, it.o + j * 128);
                ptx::tma_load_3d(sV + st * kTile + kVBox, mV, &v_full[st], 0, 2 * H + it.h, it.o + j * 128 + 64);
                ++nv;
                if (j == 0) iter.lookahead();           // while S_0 / the next k_empty are pending
            }
        }
      }
      __syncwarp();
    } else if (warp == 9) {
      {
        // ---------------- MMA issuer: the whole warp runs the loop converged and one elected
        // lane issues (warp-uniform descriptors, no per-MMA ELECT loop; umma_gemm.cu)
        const uint32_t idesc_s = ptx::idesc_bf16(128, 128, 0);
        const uint32_t idesc_o = ptx::idesc_bf16(128, 64, 1);
        const uint64_t qd = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 0, 1024);
        const uint64_t kd = ptx::smem_desc_sw128(ptx::smem_u32(sK), 0, 1024);
        uint32_t ns = 0, npv = 0, nitem = 0;
        auto issue_s = [&](int j, int nk_item) {
            if (ns > 0) ptx::mbar_wait(s_used, (ns - 1) & 1);      // softmax holds the previous S
            ptx::mbar_wait(k_full, ns & 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                ATT_TRACE(ns, 6);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    ptx::umma_bf16(tmem, qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idesc_s, kk > 0 ? 1u : 0u);
                ptx::umma_commit(s_full);
                ptx::umma_commit(k_empty);
                if (j == nk_item - 1) ptx::umma_commit(q_empty);
            }
            __syncwarp();
            ++ns;
        };
        int nk = 0;
        if ((int)blockIdx.x < n_items) {
            ptx::mbar_wait(q_full, 0);
            nk = (info[0].y + 127) / 128;
            issue_s(0, nk);
        }
        for (int k = (int)blockIdx.x; k < n_items; k += (int)gridDim.x) {
            ATT_TRACE(384 + (int)nitem, 0);
            int nk_next = 0;
            for (int j = 0; j < nk; ++j) {
                if (j + 1 < nk) {
                    issue_s(j + 1, nk);
                } else if (k + (int)gridDim.x < n_items) {
                    // the next item's first S goes to the tensor core BEFORE this item's last PV
                    // (it only needs the softmax to have pulled the last S into registers), so
                    // the softmax finds it ready when it finishes this item
                    ptx::mbar_wait(q_full, (nitem + 1) & 1);
                    ATT_TRACE(256 + (int)nitem + 1, 7);
                    nk_next = (info[(nitem + 1) & 1].y + 127) / 128;
                    issue_s(0, nk_next);
                }
                ptx::mbar_wait(p_ready, npv & 1);                       // P_j written, O rescaled
                if (j == 0 && nitem > 0) ptx::mbar_wait(o_free, (nitem - 1) & 1);   // previous O read out
                const int st = (int)(npv & 1);
                ptx::mbar_wait(&v_full[st], (npv >> 1) & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    ATT_TRACE(npv, 7);
#pragma unroll
                    for (int kb = 0; kb < 2; ++kb) {
                        const uint64_t vd = ptx::smem_desc_sw128(ptx::smem_u32(sV + st * kTile + kb * kVBox), 8192, 1024);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)        // P_j in TMEM cols [192, 256): 16 keys = 8 cols
                            umma_bf16_ts(tmem + 128, tmem + kPCol + (uint32_t)(8 * (4 * kb + kk)),
                                         vd + (uint64_t)(kk * 128), idesc_o, (j > 0 || kb > 0 || kk > 0) ? 1u : 0u);
                    }
                    ptx::umma_commit(pv_done);
                    ptx::umma_commit(&v_empty[st]);
                }
                __syncwarp();
                ++npv;
            }
            ATT_TRACE(384 + (int)nitem, 1);
            ++nitem;
            nk = nk_next;
        }
      }
      __syncwarp();
    } else {

    // ---------------- softmax warps: row q, key half `half` (64 keys) of each 128-key block
    const int quarter = (int)(warp & 3), half = (int)(warp >> 2);
    const int q = quarter * 32 + (int)lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t ns = 0, npv = 0, nitem = 0;
    for (int k = (int)blockIdx.x; k < n_items; k += (int)gridDim.x, ++nitem) {
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 0);
        ptx::mbar_wait(q_full, nitem & 1);         // the item's (o, L, qt, h) is published
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 1);
        const int4 it = info[nitem & 1];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(info_read);
        const int L = it.y, nk = (L + 127) / 128;
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < nk; ++j) {
            ptx::mbar_wait(s_full, ns & 1);
            ptx::tc_fence_after();
            const int tb = (int)ns;
            const bool tr = warp == 0 && lane == 0;
            if (tr) ATT_TRACE(tb, 0);
            float v[64];
            {
                uint32_t r[4][16];                    // four loads in flight, one wait
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld16_nowait(trow + (uint32_t)(half * 64 + c * 16), r[c]);
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_wait16(r[c]);
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[c * 16 + e] = __uint_as_float(r[c][e]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(s_used);  // the MMA warp may overwrite S now
            float *rd = red + (ns & 1) * 256;         // parity buffer: a fast half never overwrites
            ++ns;                                     // the max its partner has not read yet
            const int kbase = j * 128 + half * 64;    // key index of v[0]
            const int nvalid = min(max(L - kbase, 0), 64);   // keys of this half-block inside the request
            // a partial half-block runs the same vectorised code: keys >= L are left out of the max
            // (read as -inf) and their exponentials zeroed; a fully masked one skips the exponentials
            float mx = -INFINITY;
            if (nvalid == 64) {
                float ma = v[0], mb = v[1];
#pragma unroll
                for (int e = 2; e < 62; e += 4) {
                    ma = fmax3(ma, v[e], v[e + 1]);
                    mb = fmax3(mb, v[e + 2], v[e + 3]);
                }
                mx = fmax3(ma, mb, fmaxf(v[62], v[63]));
            } else if (nvalid > 0) {
                float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
                for (int e = 0; e < 64; e += 4) {
                    ma = fmax3(ma, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
                    mb = fmax3(mb, e + 2 < nvalid ? v[e + 2] : -INFINITY, e + 3 < nvalid ? v[e + 3] : -INFINITY);
                }
                mx = fmaxf(ma, mb);
            }
            if (tr) ATT_TRACE(tb, 1);
            rd[half * 128 + q] = mx;
            // the previous item's O tile left sP through a TMA store issued by thread 0: it must
            // have finished reading before anyone writes P_j (after this barrier)
            if (j == 0 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            ptx::named_bar_sync(1, kSoftmaxThreads);
            if (tr) ATT_TRACE(tb, 2);
            // lazy rescaling: the exponent base m_run moves only when the row max grew by more
            // than 2^kLazy in exp2 units (P then stays <= 2^kLazy, exact in fp32 / bf16 range;
            // l and O use the same base, so the final O / l is unchanged).  Both key halves of
            // a row see the same maxima, so they take the same decision.
            const float m_blk = fmaxf(rd[q], rd[128 + q]);
            const bool grow = (m_blk - m_run) * sl2 > kLazy;               // m_run = -inf: always
            const float m_new = grow ? m_blk : m_run;
            const float alpha = grow ? ptx::ex2_approx((m_run - m_new) * sl2) : 1.f;   // -inf -> 0
            const float ms = m_new * sl2;
            float2 sa = make_float2(0.f, 0.f), sb = sa;
            if (nvalid > 0) {
                const float2 sc = make_float2(sl2, sl2), nm = make_float2(-ms, -ms);
#pragma unroll
                for (int e = 0; e < 64; e += 2) {
                    float2 x = ffma2(make_float2(v[e], v[e + 1]), sc, nm);
                    if (((e >> 1) & 7) < NIMBLE_ATTN_POLY) {
                        x = exp2_poly2(x);
                    } else {
                        x.x = ptx::ex2_approx(x.x);
                        x.y = ptx::ex2_approx(x.y);
                    }
                    v[e] = x.x;
                    v[e + 1] = x.y;
                }
            }
            if (nvalid < 64) {                        // exactly 0 past L (the poly floors at 2^-125)
#pragma unroll
                for (int e = 0; e < 64; ++e) v[e] = e < nvalid ? v[e] : 0.f;
            }
#pragma unroll
            for (int e = 0; e < 64; e += 4) {
                sa = fadd2(sa, make_float2(v[e], v[e + 1]));
                sb = fadd2(sb, make_float2(v[e + 2], v[e + 3]));
            }
            sa = fadd2(sa, sb);
            l_run = l_run * alpha + (sa.x + sa.y);
            m_run = m_new;
            if (tr) ATT_TRACE(tb, 3);
            // P_{j-1} must be consumed (and O final for block j-1) before P / O are touched; at
            // j = 0 the previous item's epilogue already waited for its last PV
            if (j > 0) {
                ptx::mbar_wait(pv_done, npv & 1);
                ++npv;
                ptx::tc_fence_after();
            }
            if (tr) ATT_TRACE(tb, 4);
            // P_j as bf16 pairs into TMEM (the A operand of P.V): this row's 64 keys of the block half
            // are 32 columns of lane q, keys (2c, 2c+1) in column c
            {
                uint32_t pw[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * c], v[2 * c + 1]);
                    pw[c] = *reinterpret_cast<uint32_t *>(&h2);
                }
                tmem_st32(trow + kPCol + (uint32_t)(half * 32), pw);
            }
            // rescale this row's O half (32 of the 64 output columns) when the running max grew
            if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float t[16];
                    const uint32_t oa = trow + 128u + (uint32_t)(half * 32 + c * 16);
                    ptx::tmem_ld16(oa, t);
#pragma unroll
                    for (int e = 0; e < 16; ++e) t[e] *= alpha;
                    tmem_st16(oa, t);
                }
                tmem_st_wait();
            }
            tmem_st_wait();                           // P (tcgen05.st) complete before the MMA reads it
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(p_ready);
            if (tr) ATT_TRACE(tb, 5);
        }
        // ---------------- epilogue: O / rowsum
        redl[half * 128 + q] = l_run;
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 2);
        ptx::mbar_wait(pv_done, npv & 1);
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 3);
        ++npv;
        ptx::tc_fence_after();
        ptx::named_bar_sync(1, kSoftmaxThreads);
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 4);
        const float inv = 1.f / (redl[q] + redl[128 + q]);
        float t0[16], t1[16];                         // every lane loads: tcgen05.ld is warp-collective
        ptx::tmem_ld16(trow + 128u + (uint32_t)(half * 32), t0);
        ptx::tmem_ld16(trow + 128u + (uint32_t)(half * 32 + 16), t1);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(o_free);      // the next item's first PV may overwrite O
        if (warp == 0 && lane == 0) ATT_TRACE(448 + (int)nitem, 5);
        const int q0 = it.z * 128;
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 a = __floats2bfloat162_rn(t0[2 * e] * inv, t0[2 * e + 1] * inv);
            __nv_bfloat162 b = __floats2bfloat162_rn(t1[2 * e] * inv, t1[2 * e + 1] * inv);
            w[e] = *reinterpret_cast<uint32_t *>(&a);
            w[8 + e] = *reinterpret_cast<uint32_t *>(&b);
        }
        // stage the normalised O tile in the (now idle) P buffer in the 128-B swizzle and let
        // asynchronous TMA stores write it — the softmax warps go straight on to the next item
        // instead of waiting out 64 B of global stores per row (measured: the per-row output
        // stores cost 10 us of a 76 us layer).  A full tile is one 128-row store; a partial
        // tile's n = L - q0 valid rows leave as 64/32/16/8-row boxes (a TMA box cannot clip at
        // the request boundary L_i) plus plain stores for the last n % 8 rows.
        const int nv = min(128, L - q0);                    // valid rows of this query tile
        const int n8 = nv & ~7;                             // rows covered by TMA boxes
        if (q < n8) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = half * 4 + e;                 // 16-B chunk of the 128-B row
                *reinterpret_cast<uint4 *>(sP + q * 128 + ((c ^ (q & 7)) << 4)) =
                    make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
            }
        } else if (q < nv) {
            __nv_bfloat16 *dst = p.out + (int64_t)(it.x + q0 + q) * p.ld_out + it.w * 64 + half * 32;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                reinterpret_cast<uint4 *>(dst)[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
        }
        if (n8 > 0) {
            ptx::fence_async_smem();
            ptx::named_bar_sync(1, kSoftmaxThreads);
            if (threadIdx.x == 0) {
                if (n8 == 128) {
                    ptx::tma_store_2d(&tmO, sP, it.w * 64, it.x + q0);
                } else {
                    int r0 = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {            // box rows 64, 32, 16, 8
                        const int br = 64 >> b;
                        if (n8 & br) {
                            ptx::tma_store_2d(&tmOp.box[b], sP + r0 * 128, it.w * 64, it.x + q0 + r0);
                            r0 += br;
                        }
                    }
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        // redl is rewritten by the next item only after this item's blocks: the named barrier of
        // the next item's first block orders it after every thread's read above
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // sP read out
    }   // softmax warps
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 256);
    }
    if (trace)                                        // CTA 0's timeline -> the global trace buffer
        for (int i = threadIdx.x; i < 256 * 8; i += kThreads) {
            const int sl = i >> 3, blk = sl < 64 ? sl : sl < 128 ? sl + 192 : sl + 256;
            trace[blk * 8 + (i & 7)] = strace[i];
        }
    if (p.trace && threadIdx.x == 0) {                // per-CTA span (scripts/attn_balance.py)
        p.trace[8192 + 2 * blockIdx.x] = t_start;
        p.trace[8192 + 2 * blockIdx.x + 1] = ptx::globaltimer();
    }
}

}  // namespace

size_t attention_smem_bytes(int max_len) {
    (void)max_len;
    return kSmemBytes;
}

int attention_max_requests() { return kMaxReq; }

int attention_grid(int R, int max_len, int heads) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
    }
    const int64_t upper = (int64_t)R * ((max_len + 127) / 128) * heads;   // items, if every L_i = max_len
    const int64_t g = (int64_t)kCtasPerSm * sms;
    return (int)(upper < g ? upper : g);
}

cudaError_t launch_attention_varlen(const CUtensorMap &tmQK, const CUtensorMap &tmV, const CUtensorMap &tmO,
                                    const CUtensorMap *tmOparts, const int32_t *seq_off,
                                    int R, int max_len, int heads, float scale, __nv_bfloat16 *out, int64_t ld_out,
                                    int64_t T_max, cudaStream_t s, CUtensorMap *map_slots, bool patch_T,
                                    unsigned long long *trace) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attention_varlen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kSmemBytes);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    AttnParams p;
    p.seq_off = seq_off;
    p.R = R;
    p.heads = heads;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = out;
    p.ld_out = ld_out;
    p.map_slots = map_slots;
    p.patch_T = patch_T ? 1 : 0;
    p.T_max = (int32_t)T_max;
    p.max_len = max_len;
    p.trace = trace;
    const dim3 grid((unsigned)attention_grid(R, max_len, heads));
    OutMaps op;
    for (int b = 0; b < 4; ++b) op.box[b] = tmOparts[b];
    return launch_pdl(attention_varlen_kernel, grid, dim3(kThreads), attention_smem_bytes(max_len), s, tmQK, tmV, tmO,
                      op, p);
}

}  // namespace nimble
