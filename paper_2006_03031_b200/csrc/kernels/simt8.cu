// fp32 CUDA-core dense with the paper's residue-specialised symbolic tiling
// (Nimble §3.5): the symbolic row extent M is tiled by t = 8
// (the factor the paper's tuner chose) and rewritten M = 8k + r.
// Each CTA owns 32 output features (lane = feature, 4 warps splitting K) and one 8-row tile:
// CTAs blockIdx.y < k run the full tile with no guards; the single tail CTA
// (blockIdx.y == k) runs a loop compiled for exactly r rows (variant r, no
// guards).  The FALLBACK variant (-1) is the "fully guarded symbolic kernel":
// every row of every tile is checked against M at run time.  The static twin
// is the same body with M a compile-time constant (the paper's static codegen
// baseline, fig:sym-codegen PAPER.md:696-703).
#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kChunk = 64;               // k per warp per round
constexpr int kWarps = 4;                // the CTA's warps split K; lane = output feature
constexpr int kFeat = 32;                // output features per CTA

// ROWS >= 0: compile-time row count (no guards); ROWS < 0: runtime-guarded rows.
// CTA = 32 features x one 8-row tile; warp w takes the k-chunks w, w + 4, ... (64 wide) of
// every staged 256-wide round, and the four partial sums are added in warp order (fixed,
// deterministic).  4x the CTAs of a thread-per-feature-whole-K layout: the weight stream of a
// small-M call (LSTM input projection at T = 1, N = 2600) spreads over 4x the SMs.
template <int ROWS>
__device__ __forceinline__ void simt8_tile(const Simt8Params &p, int row0, int rows_rt) {
    __shared__ float xs[8][kWarps * kChunk];
    __shared__ float part[kWarps - 1][8][kFeat];
    const int lane = (int)threadIdx.x & 31, warp = (int)threadIdx.x >> 5;
    const int n = blockIdx.x * kFeat + lane;
    const bool n_ok = n < p.N;
    float acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.f;

    for (int k0 = 0; k0 < p.K; k0 += kWarps * kChunk) {
        __syncthreads();
        // stage the 8 x 256 x-round (rows beyond the tile / K are zeros, never read from memory)
        for (int e = threadIdx.x; e < 8 * kWarps * kChunk; e += 32 * kWarps) {
            const int r = e / (kWarps * kChunk), kk = e % (kWarps * kChunk);
            const bool live = (ROWS >= 0 ? r < ROWS : r < rows_rt) && (k0 + kk < p.K);
            xs[r][kk] = live ? p.x[(int64_t)(row0 + r) * p.ldx + k0 + kk] : 0.f;
        }
        const int kw = k0 + warp * kChunk;               // this warp's 64-wide chunk
        float w[kChunk];
        const float *wrow = p.W + (int64_t)n * p.ldw + kw;
#pragma unroll
        for (int q = 0; q < kChunk / 4; ++q) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (n_ok && kw + 4 * q < p.K) v = *reinterpret_cast<const float4 *>(wrow + 4 * q);
            w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
        }
        __syncthreads();
        const float *xw = &xs[0][warp * kChunk];
        if (ROWS >= 0) {
#pragma unroll
            for (int r = 0; r < (ROWS >= 0 ? ROWS : 0); ++r)
#pragma unroll
                for (int kk = 0; kk < kChunk; ++kk) acc[r] = fmaf(w[kk], xw[r * kWarps * kChunk + kk], acc[r]);
        } else {
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < rows_rt)                                   // the boundary check residue
#pragma unroll                                                     // specialisation removes
                    for (int kk = 0; kk < kChunk; ++kk) acc[r] = fmaf(w[kk], xw[r * kWarps * kChunk + kk], acc[r]);
        }
    }
    // partial sums of warps 1..3 -> warp 0, added in warp order
    if (warp > 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) part[warp - 1][r][lane] = acc[r];
    }
    __syncthreads();
    if (warp > 0 || !n_ok) return;
#pragma unroll
    for (int q = 0; q < kWarps - 1; ++q)
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] += part[q][r][lane];
    const float b = (p.epi >= 1) ? p.bias[n] : 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (ROWS >= 0 ? r >= ROWS : r >= rows_rt) break;
        const int64_t row = row0 + r;
        float v = acc[r] + b;
        if (p.epi == 2) v = ptx::gelu_erf(v);
        if (p.epi == 3) v += p.res[row * p.ldr + n];
        p.y[row * p.ldy + n] = v;
    }
}

// Variant TAIL in 0..7: full tiles unguarded, tail compiled for exactly TAIL rows.
template <int TAIL>
__global__ void __launch_bounds__(128) simt8_dense_kernel(const Simt8Params p) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int row0 = blockIdx.y * 8;
    if ((int)blockIdx.y < p.k_tiles) simt8_tile<8>(p, row0, 8);
    else simt8_tile<TAIL>(p, row0, TAIL);
}

// FALLBACK: every tile guarded at run time.
__global__ void __launch_bounds__(128) simt8_dense_fallback(const Simt8Params p) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int row0 = blockIdx.y * 8;
    simt8_tile<-1>(p, row0, min(8, p.M - row0));
}

// Static twin: M compile-time (k = M / 8 full tiles, tail of M % 8 rows).
template <int SM>
__global__ void __launch_bounds__(128) simt8_static_kernel(const Simt8Params p) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    constexpr int k = SM / 8, r = SM % 8;
    const int row0 = blockIdx.y * 8;
    if ((int)blockIdx.y < k) simt8_tile<8>(p, row0, 8);
    else simt8_tile<r>(p, row0, r);
}

template <int SM>
cudaError_t launch_static_rec(const Simt8Params &p, dim3 grid, cudaStream_t s) {
    if constexpr (SM > 64) {
        return cudaErrorInvalidValue;
    } else {
        if (p.M == SM) return launch_pdl(simt8_static_kernel<SM>, grid, dim3(128), 0, s, p);
        return launch_static_rec<SM + 1>(p, grid, s);
    }
}

}  // namespace

cudaError_t launch_simt8_static(const Simt8Params &p, dim3 grid, cudaStream_t s) { return launch_static_rec<1>(p, grid, s); }

cudaError_t launch_simt8(const Simt8Params &p, int variant, dim3 grid, cudaStream_t s) {
    switch (variant) {
        case 0: return launch_pdl(simt8_dense_kernel<0>, grid, dim3(128), 0, s, p);
        case 1: return launch_pdl(simt8_dense_kernel<1>, grid, dim3(128), 0, s, p);
        case 2: return launch_pdl(simt8_dense_kernel<2>, grid, dim3(128), 0, s, p);
        case 3: return launch_pdl(simt8_dense_kernel<3>, grid, dim3(128), 0, s, p);
        case 4: return launch_pdl(simt8_dense_kernel<4>, grid, dim3(128), 0, s, p);
        case 5: return launch_pdl(simt8_dense_kernel<5>, grid, dim3(128), 0, s, p);
        case 6: return launch_pdl(simt8_dense_kernel<6>, grid, dim3(128), 0, s, p);
        case 7: return launch_pdl(simt8_dense_kernel<7>, grid, dim3(128), 0, s, p);
        default: return launch_pdl(simt8_dense_fallback, grid, dim3(128), 0, s, p);
    }
}

}  // namespace nimble
