// Fused variable-length attention over token-packed requests:
// for every request i (tokens [o_i, o_i + L_i) of a packed QKV [T x 3d]) and head h,
//     C_h = softmax(Q_h K_h^T * scale) V_h
// in ONE launch, with L_i a per-request symbolic extent (PAPER.md:255 one symbol for the
// equal dynamic dims; P:575 BERT's dynamic sequence length).  It replaces the
// bmm_dyn -> softmax_rows -> bmm_dyn triple and never writes S or P to HBM.
//
// CTA = (query tile of 128, head, request), 288 threads, online softmax over 128-key blocks:
//   warp 8 lane 0  TMA producer: Q tile, then per key block K_j [128 x 64] (single buffer) and
//                  V_j (MN-major, two 64-key boxes, 2-stage ring).
//   warp 8 lane 1  MMA issuer: S = Q K_j^T into TMEM cols [0,128) as soon as the previous S
//                  has been read; O += P_j V_j into TMEM cols [128,192) once P_j is written.
//   warps 0-7      softmax: row q = TMEM lane 32*(w%4)+lane, key half (w/4) of the block held
//                  in registers; running max / sum; unnormalised P_j written as bf16 straight
//                  into the UMMA K-major swizzled smem layout; O rescaled in TMEM when the
//                  running max grows; epilogue O / rowsum -> bf16.
// TMEM 256 columns and ~99 KB smem per CTA: two CTAs share an SM.  Keys >= L_i get P = 0;
// query rows >= L_i are computed but never stored.
#include <cstdint>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kSoftmaxThreads = 256;     // warps 0-7
constexpr int kThreads = kSoftmaxThreads + 32;   // + warp 8: lane 0 TMA producer, lane 1 MMA issuer
constexpr int kTile = 128 * 64 * 2;       // Q tile / K block / V block (128 keys) / P half: 16 KiB
constexpr int kVBox = 64 * 64 * 2;        // one V TMA box (64 keys): 8 KiB
constexpr int kSmemBytes = 1024 + 6 * kTile + 2048 + 512;   // ~99 KB: two CTAs per SM

struct AttnParams {
    const int32_t *seq_off;   // [R + 1] prefix sums of request lengths (device)
    int32_t heads;
    float scale_log2;         // scale * log2(e)
    __nv_bfloat16 *out;
    int64_t ld_out;
    CUtensorMap *map_slots;   // device token count: 2 per-CTA slots for the extent-patched maps
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

__global__ void __launch_bounds__(kThreads, 2)
    attention_varlen_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                            const AttnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int qt = blockIdx.x, h = blockIdx.y, req = blockIdx.z;
    ptx::pdl_wait();                              // QKV comes from the previous kernel
    ptx::pdl_trigger();
    const int o = __ldg(p.seq_off + req);
    const int L = __ldg(p.seq_off + req + 1) - o;
    const int q0 = qt * 128;
    if (q0 >= L) return;                          // request shorter than this query tile
    const int nk = (L + 127) / 128;               // key blocks
    uint8_t *sQ = smem;
    uint8_t *sK = smem + kTile;                   // K block (single buffer: only the short S MMA reads it)
    uint8_t *sV = smem + 2 * kTile;               // [2] V blocks (two 64-key boxes each)
    uint8_t *sP = smem + 4 * kTile;               // P block: 2 x (64 keys) K-major atoms = 32 KiB
    float *red = reinterpret_cast<float *>(smem + 6 * kTile);          // [2][128] row max
    float *redl = red + 256;                                            // [2][128] row sums
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 6 * kTile + 2048);
    uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = bar + 2, *v_full = bar + 3, *v_empty = bar + 5,
             *s_full = bar + 7, *s_used = bar + 8, *p_ready = bar + 9, *pv_done = bar + 10;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 11);
    uint8_t *smaps = reinterpret_cast<uint8_t *>(bar) + 256;            // 2 x 128-B maps being patched
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmQK);
        ptx::prefetch_tmap(&tmV);
        ptx::mbar_init(q_full, 1);
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
        ptx::fence_mbar_init();
        ptx::fence_async_smem();
    }
    if (warp == 8) ptx::tmem_alloc(tmem_slot, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;             // S: cols [0,128), O: cols [128,192)

    // device token count (nimble_attention_varlen_dev): T = seq_off[R] is data, so this CTA
    // publishes copies of both maps with the token extent patched to T (rows past T then
    // zero-fill exactly as with a host-encoded T).
    const CUtensorMap *mQK = &tmQK, *mV = &tmV;
    if (p.map_slots && warp == 8) {
        const uint32_t T = (uint32_t)__ldg(p.seq_off + gridDim.z);
        CUtensorMap *slot = p.map_slots + 2 * (size_t)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
        mQK = ptx::tmap_patch_extent<2>(&tmQK, smaps, slot, T, lane);
        mV = ptx::tmap_patch_extent<2>(&tmV, smaps + 128, slot + 1, T, lane);
    }

    if (warp == 8) {
      if (lane == 0) {
        // ---------------- producer: Q once, then K_j / V_j through a 2-stage ring
        ptx::mbar_arrive_expect_tx(q_full, kTile);
        ptx::tma_load_3d(sQ, mQK, q_full, 0, h, o + q0);
        for (int j = 0; j < nk; ++j) {
            const int st = j & 1, use = j >> 1;
            if (j > 0) ptx::mbar_wait(k_empty, (j - 1) & 1);          // S_{j-1} has read K
            ptx::mbar_arrive_expect_tx(k_full, kTile);
            ptx::tma_load_3d(sK, mQK, k_full, 0, p.heads + h, o + j * 128);
            if (use > 0) ptx::mbar_wait(&v_empty[st], (use - 1) & 1); // PV_{j-2} has read V
            ptx::mbar_arrive_expect_tx(&v_full[st], kTile);
            ptx::tma_load_3d(sV + st * kTile, mV, &v_full[st], 0, 2 * p.heads + h, o + j * 128);
            ptx::tma_load_3d(sV + st * kTile + kVBox, mV, &v_full[st], 0, 2 * p.heads + h, o + j * 128 + 64);
        }
      } else if (lane == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc_s = ptx::idesc_bf16(128, 128, 0);
        const uint32_t idesc_o = ptx::idesc_bf16(128, 64, 1);
        const uint64_t qd = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 0, 1024);
        const uint64_t kd = ptx::smem_desc_sw128(ptx::smem_u32(sK), 0, 1024);
        auto issue_s = [&](int j) {
            ptx::mbar_wait(k_full, j & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                ptx::umma_bf16(tmem, qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idesc_s, kk > 0 ? 1u : 0u);
            ptx::umma_commit(s_full);
            ptx::umma_commit(k_empty);
        };
        ptx::mbar_wait(q_full, 0);
        issue_s(0);
        for (int j = 0; j < nk; ++j) {
            if (j + 1 < nk) {
                ptx::mbar_wait(s_used, j & 1);    // softmax holds S_j in registers: buffer free
                issue_s(j + 1);
            }
            ptx::mbar_wait(p_ready, j & 1);       // P_j written, O rescaled
            const int st = j & 1;
            ptx::mbar_wait(&v_full[st], (j >> 1) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int kb = 0; kb < 2; ++kb) {
                const uint64_t pd = ptx::smem_desc_sw128(ptx::smem_u32(sP + kb * kTile), 0, 1024);
                const uint64_t vd = ptx::smem_desc_sw128(ptx::smem_u32(sV + st * kTile + kb * kVBox), 8192, 1024);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    ptx::umma_bf16(tmem + 128, pd + (uint64_t)(kk * 2), vd + (uint64_t)(kk * 128), idesc_o,
                                   (j > 0 || kb > 0 || kk > 0) ? 1u : 0u);
            }
            ptx::umma_commit(pv_done);
            ptx::umma_commit(&v_empty[st]);
        }
      }
      __syncwarp();
    } else {

    // ---------------- softmax warps: row q, key half `half` (64 keys) of each 128-key block
    const int quarter = (int)(warp & 3), half = (int)(warp >> 2);
    const int q = quarter * 32 + (int)lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = p.scale_log2;
    for (int j = 0; j < nk; ++j) {
        ptx::mbar_wait(s_full, j & 1);
        ptx::tc_fence_after();
        float v[64];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float t[16];
            ptx::tmem_ld16(trow + (uint32_t)(half * 64 + c * 16), t);
#pragma unroll
            for (int e = 0; e < 16; ++e) v[c * 16 + e] = t[e];
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_used);  // the MMA warp may overwrite S now
        const int kbase = j * 128 + half * 64;    // key index of v[0]
        float mx = -INFINITY;
        if (kbase + 64 <= L) {
#pragma unroll
            for (int e = 0; e < 64; e += 4) mx = fmaxf(mx, fmaxf(fmaxf(v[e], v[e + 1]), fmaxf(v[e + 2], v[e + 3])));
        } else {
#pragma unroll
            for (int e = 0; e < 64; ++e)
                if (kbase + e < L) mx = fmaxf(mx, v[e]);
        }
        red[half * 128 + q] = mx;
        ptx::named_bar_sync(1, kSoftmaxThreads);
        const float m_new = fmaxf(m_run, fmaxf(red[q], red[128 + q]));
        const float alpha = ptx::ex2_approx((m_run - m_new) * sl2);   // m_run = -inf -> 0
        const float ms = m_new * sl2;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        if (kbase + 64 <= L) {
#pragma unroll
            for (int e = 0; e < 64; ++e) v[e] = ptx::ex2_approx(fmaf(v[e], sl2, -ms));
        } else {
#pragma unroll
            for (int e = 0; e < 64; ++e) v[e] = (kbase + e < L) ? ptx::ex2_approx(fmaf(v[e], sl2, -ms)) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 64; e += 4) { s0 += v[e]; s1 += v[e + 1]; s2 += v[e + 2]; s3 += v[e + 3]; }
        l_run = l_run * alpha + ((s0 + s1) + (s2 + s3));
        m_run = m_new;
        // P_{j-1} must be consumed (and O final for block j-1) before P / O are touched
        if (j > 0) {
            ptx::mbar_wait(pv_done, (j - 1) & 1);
            ptx::tc_fence_after();
        }
        // P_j: this warp group's 64 keys = one K-major 128-B-swizzled atom column block
        uint8_t *rowp = sP + half * kTile + q * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[c * 8 + 2 * e], v[c * 8 + 2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t *>(&h2);
            }
            *reinterpret_cast<uint4 *>(rowp + ((c ^ (q & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        // rescale this row's O half (32 of the 64 output columns) when the running max grew
        if (j > 0 && __any_sync(0xffffffffu, alpha < 1.f)) {
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
        ptx::fence_async_smem();                  // P (generic stores) -> tensor-core reads
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_ready);
    }
    // ---------------- epilogue: O / rowsum
    redl[half * 128 + q] = l_run;
    ptx::mbar_wait(pv_done, (nk - 1) & 1);
    ptx::tc_fence_after();
    ptx::named_bar_sync(1, kSoftmaxThreads);
    const float inv = 1.f / (redl[q] + redl[128 + q]);
    float t0[16], t1[16];                         // every lane loads: tcgen05.ld is warp-collective
    ptx::tmem_ld16(trow + 128u + (uint32_t)(half * 32), t0);
    ptx::tmem_ld16(trow + 128u + (uint32_t)(half * 32 + 16), t1);
    if (q0 + q < L) {
        __nv_bfloat16 *dst = p.out + (int64_t)(o + q0 + q) * p.ld_out + h * 64 + half * 32;
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 a = __floats2bfloat162_rn(t0[2 * e] * inv, t0[2 * e + 1] * inv);
            __nv_bfloat162 b = __floats2bfloat162_rn(t1[2 * e] * inv, t1[2 * e + 1] * inv);
            w[e] = *reinterpret_cast<uint32_t *>(&a);
            w[8 + e] = *reinterpret_cast<uint32_t *>(&b);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            reinterpret_cast<uint4 *>(dst)[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
    }
    }   // softmax warps
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 256);
    }
}

}  // namespace

size_t attention_smem_bytes(int max_len) {
    (void)max_len;
    return kSmemBytes;
}

cudaError_t launch_attention_varlen(const CUtensorMap &tmQK, const CUtensorMap &tmV, const int32_t *seq_off,
                                    int R, int max_len, int heads, float scale, __nv_bfloat16 *out, int64_t ld_out,
                                    cudaStream_t s, CUtensorMap *map_slots) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attention_varlen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kSmemBytes);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    AttnParams p;
    p.seq_off = seq_off;
    p.heads = heads;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = out;
    p.ld_out = ld_out;
    p.map_slots = map_slots;
    const dim3 grid((unsigned)((max_len + 127) / 128), (unsigned)heads, (unsigned)R);
    return launch_pdl(attention_varlen_kernel, grid, dim3(kThreads), attention_smem_bytes(max_len), s, tmQK, tmV, p);
}

}  // namespace nimble
