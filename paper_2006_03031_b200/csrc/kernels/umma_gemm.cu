// tcgen05 / TMEM / TMA GEMM for the symbolic-shape dense and batch_matmul of
// Nimble §3.5 on sm_100a.
//
// One CTA = one 128 x n output tile (n = UMMA N of this tile: full width, or the
// residue-specialised tail width 16*ceil(r/16) chosen by the dispatch function)
// over one K slice.  256 threads, warp roles:
//   warp 0 lane 0  TMA producer: A[128 x 64] and B[box_n x 64] bf16 tiles, 128-B
//                  swizzle, into a `stages`-deep smem ring (full/empty mbarriers).
//                  Rows beyond the symbolic extent are zero-filled by TMA bounds —
//                  the dynamic dimension is never padded in memory.  With PDL the
//                  static weight operand is fetched BEFORE griddepcontrol.wait, so
//                  the weight stream overlaps the previous kernel's tail.
//   warp 1 lane 0  MMA issuer: 4 x tcgen05.mma (K = 16) per 64-wide k-block into an
//                  fp32 accumulator in TMEM; tcgen05.commit frees each smem stage.
//   warp 2         TMEM allocation / deallocation.
//   warps 0-7      epilogue: warp w reads TMEM lane quarter (w % 4) and every other
//                  16-column chunk (w / 4); alpha / bias / GELU / residual; the tile
//                  is staged in smem in the output layout and written by ONE TMA
//                  store that clips rows beyond the symbolic extent (no guards).
// split > 1: the K slices of one tile form a thread-block cluster along z; every
// CTA parks its fp32 partial in its own smem, and CTA q reduces columns
// [q*n/split, (q+1)*n/split) over ranks 0..split-1 in order through DSMEM
// (deterministic; no atomics), then runs the epilogue on them.
#include <cstdio>
#include <cstdlib>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kThreads = 256;
constexpr int kBlockK = 64;                   // one 128-B swizzle row of bf16
constexpr int kABytes = 128 * kBlockK * 2;    // 16 KiB A stage
constexpr int kSmemLimit = 232448;            // 227 KiB opt-in per CTA
constexpr int kTailBytes = 1024;              // barriers + tmem slot

__host__ __device__ inline int b_stage_bytes(int box_n, int b_mn) {
    return b_mn ? ((box_n + 63) / 64) * (64 * kBlockK * 2) : box_n * kBlockK * 2;
}

__device__ __forceinline__ float epi_apply(const UmmaParams &p, float acc, float bias_i) {
    float v = acc * p.alpha;
    if (p.epi >= 1) v += bias_i;
    if (p.epi == 2) v = ptx::gelu_erf(v);
    return v;
}

template <int B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmOut, const UmmaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int b_bytes = b_stage_bytes(p.box_n, B_MN);
    const int stage_bytes = kABytes + b_bytes;
    const int ring_bytes = p.stages * stage_bytes;
    const int red_bytes = 128 * p.box_n * ((p.split > 1 || p.out_f32) ? 4 : 2);   // epilogue staging
    uint8_t *tail = smem + (ring_bytes > red_bytes ? ring_bytes : red_bytes);
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(tail);
    uint64_t *empty_bar = full_bar + p.stages;
    uint64_t *tmem_full = empty_bar + p.stages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    const int m_tile = blockIdx.x;
    const int n_tile = blockIdx.y;
    const int split_q = blockIdx.z % p.split;
    const int batch = blockIdx.z / p.split;
    const bool last_n = (n_tile == p.n_tiles - 1);
    const int n_this = last_n ? p.n_tail : p.n_full;     // UMMA N of this tile (runtime idesc field)
    const uint32_t tmem_cols = n_this <= 32 ? 32 : n_this <= 64 ? 64 : n_this <= 128 ? 128 : 256;
    const int kb0 = (int)((int64_t)split_q * p.kb_total / p.split);
    const int kb1 = (int)((int64_t)(split_q + 1) * p.kb_total / p.split);

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        if (p.tma_store) ptx::prefetch_tmap(&tmOut);
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::fence_mbar_init();
        ptx::fence_async_smem();
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, tmem_cols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();                               // the next kernel's prologue may start now

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        const int32_t a_row = m_tile * 128;
        const int32_t b_row = n_tile * p.n_full;
        const int32_t ab = p.a_bcast ? 0 : batch;
        const int32_t bb = p.b_bcast ? 0 : batch;
        const uint32_t tx = kABytes + b_bytes;
        auto load_a = [&](int stage, int kb) {
            uint8_t *sa = smem + stage * stage_bytes;
            const int32_t kc = kb * kBlockK;
            if (p.a_batch_mid) ptx::tma_load_3d(sa, &tmA, &full_bar[stage], kc, ab, a_row);
            else ptx::tma_load_3d(sa, &tmA, &full_bar[stage], kc, a_row, ab);
        };
        auto load_b = [&](int stage, int kb) {
            uint8_t *sb = smem + stage * stage_bytes + kABytes;
            const int32_t kc = kb * kBlockK;
            if (B_MN) {
                const int chunks = (p.box_n + 63) / 64;
                for (int c = 0; c < chunks; ++c) {
                    if (p.b_batch_mid) ptx::tma_load_3d(sb + c * 8192, &tmB, &full_bar[stage], b_row + 64 * c, bb, kc);
                    else ptx::tma_load_3d(sb + c * 8192, &tmB, &full_bar[stage], b_row + 64 * c, kc, bb);
                }
            } else {
                if (p.b_batch_mid) ptx::tma_load_3d(sb, &tmB, &full_bar[stage], kc, bb, b_row);
                else ptx::tma_load_3d(sb, &tmB, &full_bar[stage], kc, b_row, bb);
            }
        };
        // prologue: the first `stages` k-blocks; static weights go out before the PDL wait
        const int npre = min(p.stages, kb1 - kb0);
        for (int s = 0; s < npre; ++s) {
            ptx::mbar_arrive_expect_tx(&full_bar[s], tx);
            if (p.a_static) load_a(s, kb0 + s);
        }
        ptx::pdl_wait();                              // producer grid's activations now visible
        for (int s = 0; s < npre; ++s) {
            if (!p.a_static) load_a(s, kb0 + s);
            load_b(s, kb0 + s);
        }
        int stage = npre % p.stages;
        uint32_t phase = (npre == p.stages) ? 1u : 0u;
        for (int kb = kb0 + npre; kb < kb1; ++kb) {
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full_bar[stage], tx);
            load_a(stage, kb);
            load_b(stage, kb);
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer (single thread)
        const uint32_t idesc = ptx::idesc_bf16(128, (uint32_t)n_this, B_MN);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const uint32_t sa = ptx::smem_u32(smem + stage * stage_bytes);
            const uint32_t sb = sa + kABytes;
            const uint64_t adesc = ptx::smem_desc_sw128(sa, 0, 1024);
            // K-major B: 8-row groups 1024 B apart.  MN-major B: 64-column chunks
            // 8 KiB apart (LBO), 8-row k groups 1024 B apart (SBO).
            const uint64_t bdesc = B_MN ? ptx::smem_desc_sw128(sb, 8192, 1024) : ptx::smem_desc_sw128(sb, 0, 1024);
#pragma unroll
            for (int kk = 0; kk < kBlockK / 16; ++kk) {
                const uint64_t a_k = adesc + (uint64_t)((kk * 32) >> 4);                // +32 B along K in the row
                const uint64_t b_k = bdesc + (uint64_t)(B_MN ? ((kk * 2048) >> 4) : ((kk * 32) >> 4));
                ptx::umma_bf16(tmem_base, a_k, b_k, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            }
            ptx::umma_commit(&empty_bar[stage]);       // smem stage free once these MMAs retire
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(tmem_full);                   // accumulator complete
    }
    __syncwarp();
    ptx::pdl_wait();                                   // epilogue reads residual / writes output

    // ---------------- epilogue: warp w owns TMEM lanes 32*(w%4).. and chunks c = w/4 (mod 2)
    ptx::mbar_wait(tmem_full, 0);
    ptx::tc_fence_after();

    const int quarter = (int)(warp & 3);
    const int half = (int)(warp >> 2);
    const int row_local = quarter * 32 + (int)lane;
    const int i = m_tile * 128 + row_local;                 // UMMA-M index
    const int j0 = n_tile * p.n_full;                       // first UMMA-N index of the tile
    const bool row_ok = i < p.rows_a;
    const int64_t out_b = (int64_t)batch * p.stride_out;
    const uint32_t tmem_row = tmem_base + ((uint32_t)(quarter * 32) << 16);
    float bias_i = 0.f;
    if (p.epi >= 1 && row_ok) bias_i = p.bias[i];
    const int n_valid = min(n_this, p.rows_b - j0);         // columns holding real data

    if (p.split == 1) {
        if (p.transposed) {
            // stage out^T tile as [n][128] in smem (lane = i -> conflict-free), then one TMA store
            for (int c0 = half * 16; c0 < n_this; c0 += 32) {
                float v[16];
                ptx::tmem_ld16(tmem_row + (uint32_t)c0, v);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int jl = c0 + q;
                    float val = epi_apply(p, v[q], bias_i);
                    if (p.epi == 3 && row_ok && jl < n_valid)
                        val += __bfloat162float(static_cast<const __nv_bfloat16 *>(p.res)[(int64_t)(j0 + jl) * p.ld_res + i]);
                    if (p.out_f32) reinterpret_cast<float *>(smem)[jl * 128 + row_local] = val;
                    else reinterpret_cast<__nv_bfloat16 *>(smem)[jl * 128 + row_local] = __float2bfloat16_rn(val);
                }
            }
            ptx::fence_async_smem();
            ptx::named_bar_sync(1, kThreads);
            if (threadIdx.x == 0) {
                if (p.out_batch_mid) ptx::tma_store_3d(&tmOut, smem, m_tile * 128, batch, j0);
                else ptx::tma_store_3d(&tmOut, smem, m_tile * 128, j0, batch);
                ptx::tma_store_commit_wait();
            }
        } else {
            // direct row-major store: thread owns row i, 16 consecutive columns per chunk
            for (int c0 = half * 16; c0 < n_this; c0 += 32) {
                float v[16];
                ptx::tmem_ld16(tmem_row + (uint32_t)c0, v);
                if (!row_ok || c0 >= n_valid) continue;
                const int64_t base = out_b + (int64_t)i * p.ld_out + j0 + c0;
                if (c0 + 16 <= n_valid) {
                    if (p.out_f32) {
                        float4 *dst = reinterpret_cast<float4 *>(static_cast<float *>(p.out) + base);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            dst[q] = make_float4(v[4 * q] * p.alpha, v[4 * q + 1] * p.alpha, v[4 * q + 2] * p.alpha,
                                                 v[4 * q + 3] * p.alpha);
                    } else {
                        uint32_t w[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * q] * p.alpha, v[2 * q + 1] * p.alpha);
                            w[q] = *reinterpret_cast<uint32_t *>(&h2);
                        }
                        uint4 *dst = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.out) + base);
                        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (c0 + q < n_valid) {
                            if (p.out_f32) static_cast<float *>(p.out)[base + q] = v[q] * p.alpha;
                            else static_cast<__nv_bfloat16 *>(p.out)[base + q] = __float2bfloat16_rn(v[q] * p.alpha);
                        }
                    }
                }
            }
        }
    } else {
        // ---------------- split-K: park the fp32 partial in own smem as red[col][128]
        float *red = reinterpret_cast<float *>(smem);
        for (int c0 = half * 16; c0 < n_this; c0 += 32) {
            float v[16];
            ptx::tmem_ld16(tmem_row + (uint32_t)c0, v);
#pragma unroll
            for (int q = 0; q < 16; ++q) red[(c0 + q) * 128 + row_local] = v[q];
        }
        ptx::cluster_sync();
        const uint32_t rank = ptx::cluster_ctarank();
        const int per = n_this / p.split;
        const int cbeg = (int)rank * per;
        uint32_t rbase[8];
        const uint32_t red_s = ptx::smem_u32(red);
#pragma unroll
        for (int r = 0; r < 8; ++r) rbase[r] = (r < p.split) ? ptx::map_shared_rank(red_s, (uint32_t)r) : 0u;
        for (int jl = cbeg + half; jl < cbeg + per; jl += 2) {
            const uint32_t off = (uint32_t)((jl * 128 + row_local) * 4);
            float part[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) part[r] = (r < p.split) ? ptx::ld_dsmem_f32(rbase[r] + off) : 0.f;
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < 8; ++r) acc += part[r];       // fixed rank order: deterministic
            if (!row_ok || jl >= n_valid) continue;
            const int64_t j = j0 + jl;
            if (p.transposed) {
                float val = epi_apply(p, acc, bias_i);
                if (p.epi == 3) val += __bfloat162float(static_cast<const __nv_bfloat16 *>(p.res)[j * p.ld_res + i]);
                const int64_t o = out_b + j * p.ld_out + i;
                if (p.out_f32) static_cast<float *>(p.out)[o] = val;
                else static_cast<__nv_bfloat16 *>(p.out)[o] = __float2bfloat16_rn(val);
            } else {
                const int64_t o = out_b + (int64_t)i * p.ld_out + j;
                if (p.out_f32) static_cast<float *>(p.out)[o] = acc * p.alpha;
                else static_cast<__nv_bfloat16 *>(p.out)[o] = __float2bfloat16_rn(acc * p.alpha);
            }
        }
        ptx::cluster_sync();                                   // keep smem alive for peers
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, tmem_cols);
    }
}

}  // namespace

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("NIMBLE_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int umma_max_stages(int box_n, int b_mn_major) {
    const int stage = kABytes + b_stage_bytes(box_n, b_mn_major);
    return (kSmemLimit - 1024 - kTailBytes) / stage;
}

size_t umma_smem_bytes(int box_n, int b_mn_major, int stages, int split, int out_bytes) {
    const size_t ring = (size_t)stages * (kABytes + b_stage_bytes(box_n, b_mn_major));
    const size_t red = (size_t)128 * box_n * (split > 1 ? 4 : out_bytes);
    return 1024 /* alignment slack */ + (ring > red ? ring : red) + kTailBytes;
}

cudaError_t launch_umma_gemm(const UmmaLaunch &L) {
    static bool attr_set[2] = {false, false};
    const void *fn = L.b_mn_major ? (const void *)umma_gemm_kernel<1> : (const void *)umma_gemm_kernel<0>;
    if (!attr_set[L.b_mn_major]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
        if (e != cudaSuccess) return e;
        attr_set[L.b_mn_major] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = L.grid;
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = L.smem_bytes;
    cfg.stream = L.stream;
    cudaLaunchAttribute attr[2];
    cfg.attrs = attr;
    cfg.numAttrs = 0;
    if (L.p.split > 1) {
        attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
        attr[cfg.numAttrs].val.clusterDim.x = 1;
        attr[cfg.numAttrs].val.clusterDim.y = 1;
        attr[cfg.numAttrs].val.clusterDim.z = (unsigned)L.p.split;
        cfg.numAttrs++;
    }
    if (pdl_enabled()) {
        attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs++;
    }
    if (L.b_mn_major) return cudaLaunchKernelEx(&cfg, umma_gemm_kernel<1>, L.tmA, L.tmB, L.tmOut, L.p);
    return cudaLaunchKernelEx(&cfg, umma_gemm_kernel<0>, L.tmA, L.tmB, L.tmOut, L.p);
}

}  // namespace nimble
