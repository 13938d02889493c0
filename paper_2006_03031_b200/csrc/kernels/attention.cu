// Fused variable-length attention over token-packed requests:
// for every request i (tokens [o_i, o_i + L_i) of a packed QKV [T x 3d]) and head h,
//     C_h = softmax(Q_h K_h^T * scale) V_h
// in ONE launch, with L_i a per-request symbolic extent (PAPER.md:255 one symbol for the
// equal dynamic dims; P:575 BERT's dynamic sequence length).  It replaces the
// bmm_dyn -> softmax_rows -> bmm_dyn triple and never writes S or P to HBM.
//
// CTA = (query tile of 128, head, request).  256 threads.
//   warp 0 lane 0  TMA producer: Q tile [128 x 64] and all key tiles K[128 x 64] of the
//                  request (128-B swizzle); after S is computed, the V blocks [64 x 64]
//                  (MN-major operand) into the same smem.
//   warp 1 lane 0  MMA issuer: S_kt = Q K_kt^T into TMEM columns [128 kt, 128 kt + 128),
//                  then O = P V into TMEM columns [0, 64) (after S has been read).
//   warps 0-7      softmax: warp w owns TMEM lanes 32*(w%4).. (query rows) and every other
//                  16-column chunk (w/4); two passes over the row in TMEM (max, then exp2 /
//                  sum, combined across the two warpgroups through smem), unnormalised P
//                  written as bf16 straight into the UMMA K-major swizzled smem layout;
//                  epilogue O / rowsum -> bf16.
// Keys >= L_i (the next request's rows, or TMA zero-fill past T) get P = 0; query rows
// >= L_i are computed but never stored.
#include <cstdint>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kThreads = 256;    // 8 warps: two warpgroups split every row's columns
constexpr int kQBytes = 128 * 64 * 2;     // Q tile / one K tile: 16 KiB
constexpr int kVBytes = 64 * 64 * 2;      // one V block (64 keys): 8 KiB
constexpr int kPBlock = 128 * 64 * 2;     // one P k-block (64 keys): 16 KiB

struct AttnParams {
    const int32_t *seq_off;   // [R + 1] prefix sums of request lengths (device)
    int32_t heads;
    float scale_log2;         // scale * log2(e)
    __nv_bfloat16 *out;
    int64_t ld_out;
    int32_t max_tiles;        // ceil(max_len / 128)
};

__global__ void __launch_bounds__(kThreads)
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
    const int nk = (L + 127) / 128;               // key tiles
    const int nkb = (L + 63) / 64;                // 64-key blocks
    // smem: region A = Q + K tiles (later V blocks), region P = P k-blocks, then barriers
    uint8_t *sQ = smem;
    uint8_t *sK = smem + kQBytes;
    uint8_t *sV = smem;                           // reuses Q/K after S is complete
    uint8_t *sP = smem + kQBytes + p.max_tiles * kQBytes;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sP + p.max_tiles * 2 * kPBlock);
    uint64_t *bar_qk = bar, *bar_s = bar + 1, *bar_v = bar + 2, *bar_o = bar + 3;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 4);
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const uint32_t tcols = nk <= 1 ? 128 : nk <= 2 ? 256 : 512;

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmQK);
        ptx::prefetch_tmap(&tmV);
        for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_mbar_init();
        ptx::fence_async_smem();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, tcols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (threadIdx.x == 0) {
        // Q tile + every key tile of this request (rows beyond T are zero-filled)
        ptx::mbar_arrive_expect_tx(bar_qk, (uint32_t)(kQBytes * (1 + nk)));
        ptx::tma_load_3d(sQ, &tmQK, bar_qk, 0, h, o + q0);
        for (int kt = 0; kt < nk; ++kt) ptx::tma_load_3d(sK + kt * kQBytes, &tmQK, bar_qk, 0, p.heads + h, o + kt * 128);
    }
    if (threadIdx.x == 32) {
        // S_kt = Q K_kt^T  (M = 128 queries, N = 128 keys, K = 64)
        ptx::mbar_wait(bar_qk, 0);
        ptx::tc_fence_after();
        const uint32_t idesc = ptx::idesc_bf16(128, 128, 0);
        const uint64_t qd = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 0, 1024);
        for (int kt = 0; kt < nk; ++kt) {
            const uint64_t kd = ptx::smem_desc_sw128(ptx::smem_u32(sK + kt * kQBytes), 0, 1024);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                ptx::umma_bf16(tmem + (uint32_t)(kt * 128), qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idesc,
                               kk > 0 ? 1u : 0u);
        }
        ptx::umma_commit(bar_s);
    }
    if (threadIdx.x == 0) {
        // V blocks into the Q/K region once the S MMAs have consumed it
        ptx::mbar_wait(bar_s, 0);
        ptx::mbar_arrive_expect_tx(bar_v, (uint32_t)(kVBytes * nkb));
        for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_3d(sV + kb * kVBytes, &tmV, bar_v, 0, 2 * p.heads + h, o + kb * 64);
    }
    __syncwarp();

    // ---------------- softmax: row q = TMEM lane 32*(warp%4) + lane, column chunks alternate by warp/4
    const int quarter = (int)(warp & 3), half = (int)(warp >> 2);
    const int q = quarter * 32 + (int)lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    float *red = reinterpret_cast<float *>(tmem_slot + 4);      // [2][128] partial max, then sum
    ptx::mbar_wait(bar_s, 0);
    ptx::tc_fence_after();
    // pass 1: row max.  Interior chunks (all 16 keys < L) take an unmasked path.
    float mx = -INFINITY;
    for (int c0 = half * 16; c0 < nk * 128; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(trow + (uint32_t)c0, v);
        if (c0 + 16 <= L) {
            float m0 = fmaxf(v[0], v[1]), m1 = fmaxf(v[2], v[3]), m2 = fmaxf(v[4], v[5]), m3 = fmaxf(v[6], v[7]);
            m0 = fmaxf(m0, fmaxf(v[8], v[9])); m1 = fmaxf(m1, fmaxf(v[10], v[11]));
            m2 = fmaxf(m2, fmaxf(v[12], v[13])); m3 = fmaxf(m3, fmaxf(v[14], v[15]));
            mx = fmaxf(mx, fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)));
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (c0 + e < L) mx = fmaxf(mx, v[e]);
        }
    }
    red[half * 128 + q] = mx;
    __syncthreads();
    mx = fmaxf(red[q], red[128 + q]);
    const float mx_s = mx * p.scale_log2;
    // pass 2: p = 2^(s*scale*log2e - max*scale*log2e) (one FFMA + one MUFU.EX2 per key),
    // four independent partial sums, bf16 pairs packed straight into the swizzled P layout.
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    for (int c0 = half * 16; c0 < nkb * 64; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(trow + (uint32_t)c0, v);
        if (c0 + 16 <= L) {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = ptx::ex2_approx(fmaf(v[e], p.scale_log2, -mx_s));
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = (c0 + e < L) ? ptx::ex2_approx(fmaf(v[e], p.scale_log2, -mx_s)) : 0.f;
        }
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
            s0 += v[e]; s1 += v[e + 1]; s2 += v[e + 2]; s3 += v[e + 3];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            w[e] = *reinterpret_cast<uint32_t *>(&h2);
        }
        // UMMA K-major SW128 layout: block kb = 64 keys, row q at 128 B, 16-B chunk c ^ (q & 7)
        const int kb = c0 >> 6, c = (c0 & 63) >> 3;
        uint8_t *rowp = sP + kb * kPBlock + q * 128;
        *reinterpret_cast<uint4 *>(rowp + (((c) ^ (q & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4 *>(rowp + (((c + 1) ^ (q & 7)) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
    }
    const float sum = (s0 + s1) + (s2 + s3);
    __syncthreads();                              // everyone has read red[] (max) before reuse
    red[half * 128 + q] = sum;
    ptx::fence_async_smem();                      // P (generic stores) -> tensor-core reads
    ptx::tc_fence_before();                       // all S reads done before O overwrites cols 0..63
    __syncthreads();

    if (threadIdx.x == 32) {
        // O = P V  (M = 128 queries, N = 64, K = keys; V MN-major)
        ptx::tc_fence_after();
        ptx::mbar_wait(bar_v, 0);
        const uint32_t idesc = ptx::idesc_bf16(128, 64, 1);
        for (int kb = 0; kb < nkb; ++kb) {
            const uint64_t pd = ptx::smem_desc_sw128(ptx::smem_u32(sP + kb * kPBlock), 0, 1024);
            const uint64_t vd = ptx::smem_desc_sw128(ptx::smem_u32(sV + kb * kVBytes), 8192, 1024);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                ptx::umma_bf16(tmem, pd + (uint64_t)(kk * 2), vd + (uint64_t)(kk * 128), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::umma_commit(bar_o);
    }
    __syncwarp();
    ptx::mbar_wait(bar_o, 0);
    ptx::tc_fence_after();
    const float inv = 1.f / (red[q] + red[128 + q]);
    const bool live = q0 + q < L;
    __nv_bfloat16 *dst = p.out + (int64_t)(o + q0 + q) * p.ld_out + h * 64;
#pragma unroll
    for (int c0 = half * 16; c0 < 64; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(trow + (uint32_t)c0, v);
        if (live) {
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * e] * inv, v[2 * e + 1] * inv);
                w[e] = *reinterpret_cast<uint32_t *>(&h2);
            }
            reinterpret_cast<uint4 *>(dst + c0)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4 *>(dst + c0)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, tcols);
    }
}

}  // namespace

size_t attention_smem_bytes(int max_len) {
    const int mt = (max_len + 127) / 128;
    return 1024 + (size_t)kQBytes * (1 + mt) + (size_t)mt * 2 * kPBlock + 64 + 2 * 128 * 4;
}

cudaError_t launch_attention_varlen(const CUtensorMap &tmQK, const CUtensorMap &tmV, const int32_t *seq_off,
                                    int R, int max_len, int heads, float scale, __nv_bfloat16 *out, int64_t ld_out,
                                    cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attention_varlen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             232448);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    AttnParams p;
    p.seq_off = seq_off;
    p.heads = heads;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = out;
    p.ld_out = ld_out;
    p.max_tiles = (max_len + 127) / 128;
    const dim3 grid((unsigned)p.max_tiles, (unsigned)heads, (unsigned)R);
    return launch_pdl(attention_varlen_kernel, grid, dim3(kThreads), attention_smem_bytes(max_len), s, tmQK, tmV, p);
}

}  // namespace nimble
