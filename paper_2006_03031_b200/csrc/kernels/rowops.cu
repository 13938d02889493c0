// Row ops around bmm_dyn in a BERT encoder layer: softmax over the dynamic
// sequence length L and LayerNorm (the paper is silent on both; DESIGN.md
// readings 9-10).  Memory-bound; 16-B vector loads where the layout allows.
#include <cstdlib>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp per row; the row is held in registers (L <= 32 * kMaxPerLane).
constexpr int kMaxPerLane = 32;   // L <= 1024

__global__ void __launch_bounds__(256) softmax_rows_kernel(const float *__restrict__ S, int64_t ldS, int64_t strideS,
                                                           __nv_bfloat16 *__restrict__ P, int64_t ldP,
                                                           int64_t strideP, int64_t batch, int64_t rows, int L) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (gw >= batch * rows) return;
    const int lane = threadIdx.x & 31;
    const int64_t b = gw / rows, i = gw % rows;
    const float *s = S + b * strideS + i * ldS;
    __nv_bfloat16 *pr = P + b * strideP + i * ldP;
    float v[kMaxPerLane];
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < kMaxPerLane; ++q) {
        const int j = lane + 32 * q;
        v[q] = (j < L) ? s[j] : -INFINITY;
        mx = fmaxf(mx, v[q]);
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < kMaxPerLane; ++q) {
        const int j = lane + 32 * q;
        v[q] = (j < L) ? __expf(v[q] - mx) : 0.f;
        sum += v[q];
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
#pragma unroll
    for (int q = 0; q < kMaxPerLane; ++q) {
        const int j = lane + 32 * q;
        if (j < L) pr[j] = __float2bfloat16_rn(v[q] * inv);
    }
    for (int64_t j = L + lane; j < ldP; j += 32) pr[j] = __float2bfloat16_rn(0.f);
}

// One warp per row, 8 rows per 256-thread CTA; lane l holds the 8-element chunks
// l, l+32, l+64, ... of its row in registers (d <= 256 * CH, d % 8 == 0), so the two
// statistics passes are register-only with warp-shuffle reductions (no __syncthreads).
template <int CH>
__global__ void __launch_bounds__(256) layernorm_warp_kernel(const __nv_bfloat16 *__restrict__ X, int64_t ldx,
                                                             const float *__restrict__ g, const float *__restrict__ be,
                                                             float eps, __nv_bfloat16 *__restrict__ Y, int64_t ldy,
                                                             int64_t rows, int d, const int32_t *__restrict__ rows_dev) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (rows_dev) {                      // device extent: the grid covers the bound `rows`
        const int32_t r = *rows_dev;
        if (r < 1 || r > rows) __trap();
        rows = r;
    }
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    const __nv_bfloat16 *x = X + row * ldx;
    float v[CH * 8];
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int j = (lane + 32 * q) * 8;
        if (j < d) {
            const uint4 u = *reinterpret_cast<const uint4 *>(x + j);
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                v[8 * q + 2 * e] = f.x;
                v[8 * q + 2 * e + 1] = f.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[8 * q + e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[8 * q + e];
    }
    const float mean = warp_sum(s) / (float)d;
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int j = (lane + 32 * q) * 8;
        if (j < d) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float t = v[8 * q + e] - mean;
                ss += t * t;
            }
        }
    }
    const float inv = rsqrtf(warp_sum(ss) / (float)d + eps);
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int j = (lane + 32 * q) * 8;
        if (j < d) {
            const float4 g0 = *reinterpret_cast<const float4 *>(g + j), g1 = *reinterpret_cast<const float4 *>(g + j + 4);
            const float4 b0 = *reinterpret_cast<const float4 *>(be + j), b1 = *reinterpret_cast<const float4 *>(be + j + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn((v[8 * q + 2 * e] - mean) * inv * gg[2 * e] + bb[2 * e],
                                                          (v[8 * q + 2 * e + 1] - mean) * inv * gg[2 * e + 1] + bb[2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t *>(&h2);
            }
            *reinterpret_cast<uint4 *>(Y + row * ldy + j) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// d = 1024 (BERT-large) at many rows: one wave of 12-warp CTAs (one per SM), each warp
// normalising `rpw` consecutive rows with gamma / beta held in registers (loaded once per warp
// instead of once per row: 8 KB of L1 traffic per row saved) and the next row's 16-B loads
// issued before the current row's arithmetic.  Per row the arithmetic is exactly
// layernorm_warp_kernel<4>'s (same order), so both agree bit for bit.
constexpr int kLnWarps = 12;
__global__ void __launch_bounds__(32 * kLnWarps, 1) layernorm_rows_kernel(const __nv_bfloat16 *__restrict__ X,
                                                                         int64_t ldx, const float *__restrict__ g,
                                                                         const float *__restrict__ be, float eps,
                                                                         __nv_bfloat16 *__restrict__ Y, int64_t ldy,
                                                                         int64_t rows, int32_t rpw,
                                                                         const int32_t *__restrict__ rows_dev) {
    constexpr int CH = 4, d = 1024;
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (rows_dev) {
        const int32_t r = *rows_dev;
        if (r < 1 || r > rows) __trap();
        rows = r;
    }
    const int64_t row0 = ((int64_t)blockIdx.x * kLnWarps + (threadIdx.x >> 5)) * rpw;
    if (row0 >= rows) return;
    const int lane = threadIdx.x & 31;
    float gg[CH * 8], bb[CH * 8];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int j = (lane + 32 * q) * 8;
        const float4 g0 = *reinterpret_cast<const float4 *>(g + j), g1 = *reinterpret_cast<const float4 *>(g + j + 4);
        const float4 b0 = *reinterpret_cast<const float4 *>(be + j), b1 = *reinterpret_cast<const float4 *>(be + j + 4);
        gg[8 * q + 0] = g0.x; gg[8 * q + 1] = g0.y; gg[8 * q + 2] = g0.z; gg[8 * q + 3] = g0.w;
        gg[8 * q + 4] = g1.x; gg[8 * q + 5] = g1.y; gg[8 * q + 6] = g1.z; gg[8 * q + 7] = g1.w;
        bb[8 * q + 0] = b0.x; bb[8 * q + 1] = b0.y; bb[8 * q + 2] = b0.z; bb[8 * q + 3] = b0.w;
        bb[8 * q + 4] = b1.x; bb[8 * q + 5] = b1.y; bb[8 * q + 6] = b1.z; bb[8 * q + 7] = b1.w;
    }
    uint4 cur[CH], nxt[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) cur[q] = *reinterpret_cast<const uint4 *>(X + row0 * ldx + (lane + 32 * q) * 8);
#pragma unroll 1
    for (int r = 0; r < rpw; ++r) {
        const int64_t row = row0 + r;
        if (row >= rows) break;
        const bool more = r + 1 < rpw && row + 1 < rows;
        if (more) {
#pragma unroll
            for (int q = 0; q < CH; ++q) nxt[q] = *reinterpret_cast<const uint4 *>(X + (row + 1) * ldx + (lane + 32 * q) * 8);
        }
        // the row stays packed (bf16) in cur[]: values are re-expanded per pass (fewer registers)
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&cur[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                sum += f.x;
                sum += f.y;
            }
        }
        const float mean = warp_sum(sum) / (float)d;
        float ss = 0.f;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&cur[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                const float t0 = f.x - mean, t1 = f.y - mean;
                ss += t0 * t0;
                ss += t1 * t1;
            }
        }
        const float inv = rsqrtf(warp_sum(ss) / (float)d + eps);
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&cur[q]);
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn((f.x - mean) * inv * gg[8 * q + 2 * e] + bb[8 * q + 2 * e],
                                                          (f.y - mean) * inv * gg[8 * q + 2 * e + 1] + bb[8 * q + 2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t *>(&h2);
            }
            *reinterpret_cast<uint4 *>(Y + row * ldy + (lane + 32 * q) * 8) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (more) {
#pragma unroll
            for (int q = 0; q < CH; ++q) cur[q] = nxt[q];
        }
    }
}

}  // namespace

cudaError_t launch_softmax_rows(const float *S, int64_t ldS, int64_t strideS, __nv_bfloat16 *P, int64_t ldP,
                                int64_t strideP, int64_t batch, int64_t rows, int64_t L, cudaStream_t s) {
    if (L > 32 * kMaxPerLane) return cudaErrorInvalidValue;
    const int64_t warps = batch * rows;
    return launch_pdl(softmax_rows_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, s, S, ldS, strideS, P, ldP,
                      strideP, batch, rows, (int)L);
}

cudaError_t launch_layernorm(const __nv_bfloat16 *X, int64_t ldx, const float *g, const float *b, float eps,
                             __nv_bfloat16 *Y, int64_t ldy, int64_t rows, int64_t d, cudaStream_t s,
                             const int32_t *rows_dev) {
    if (d > 4096 || d % 8) return cudaErrorInvalidValue;
    static const bool rows_off = [] { const char *e = std::getenv("NIMBLE_LN_ROWS"); return e && e[0] == '0'; }();
    if (d == 1024 && rows >= 4 * kLnWarps * 148 && !rows_off) {   // >= 4 rows per warp amortise gamma / beta
        const int64_t warps = (int64_t)kLnWarps * 148;
        const int32_t rpw = (int32_t)((rows + warps - 1) / warps);
        const int64_t ctas = ((rows + rpw - 1) / rpw + kLnWarps - 1) / kLnWarps;
        return launch_pdl(layernorm_rows_kernel, dim3((unsigned)ctas), dim3(32 * kLnWarps), 0, s, X, ldx, g, b, eps, Y,
                          ldy, rows, rpw, rows_dev);
    }
    const dim3 grid((unsigned)((rows + 7) / 8)), block(256);
    if (d <= 1024)
        return launch_pdl(layernorm_warp_kernel<4>, grid, block, 0, s, X, ldx, g, b, eps, Y, ldy, rows, (int)d, rows_dev);
    if (d <= 2048)
        return launch_pdl(layernorm_warp_kernel<8>, grid, block, 0, s, X, ldx, g, b, eps, Y, ldy, rows, (int)d, rows_dev);
    return launch_pdl(layernorm_warp_kernel<16>, grid, block, 0, s, X, ldx, g, b, eps, Y, ldy, rows, (int)d, rows_dev);
}

}  // namespace nimble
