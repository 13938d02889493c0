// One level of a level-batched binary Tree-LSTM (Nimble's Tree-LSTM benchmark,
// PAPER.md:575-576): the recursion over the tree ADT becomes a
// host schedule of levels (node height), and each level is one dense over the
// level's M nodes (M symbolic) with the Tree-LSTM cell fused into the epilogue.
// The epilogue writes h / c into the parent's input row so the next level
// needs no gather.  fp32, CUDA cores (each level is a few hundred kFLOP per node:
// latency-bound).
#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kNodes = 8;     // node tile (the symbolic M dimension), t = 8 as in SIMT8
constexpr int kUnits = 32;    // hidden units per CTA
constexpr int kKc = 32;       // K chunk

template <int G>
__global__ void __launch_bounds__(kNodes * kUnits) treelstm_level_kernel(const TreeParams p) {
    __shared__ float As[kNodes][kKc];
    __shared__ float Ws[G][kUnits][kKc + 1];
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int r = threadIdx.x >> 5;            // node within the tile (warp-uniform)
    const int u = threadIdx.x & 31;            // hidden unit within the tile
    const int m = blockIdx.y * kNodes + r;
    const int j = blockIdx.x * kUnits + u;
    const bool live = (m < p.M) && (j < p.H);
    const int H = p.H;
    int64_t arow = -1;
    if (m < p.M) arow = p.a_rows[m];
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.f;

    for (int k0 = 0; k0 < p.K; k0 += kKc) {
        __syncthreads();
        {
            const int kk = threadIdx.x & 31;
            As[r][kk] = (arow >= 0 && k0 + kk < p.K) ? p.A[arow * p.lda + k0 + kk] : 0.f;
        }
        for (int e = threadIdx.x; e < G * kUnits * kKc; e += kNodes * kUnits) {
            const int kk = e % kKc, row = e / kKc;
            const int g = row / kUnits, uu = row % kUnits;
            const int jj = blockIdx.x * kUnits + uu;
            Ws[g][uu][kk] = (jj < H && k0 + kk < p.K) ? p.W[(int64_t)(g * H + jj) * p.ldw + k0 + kk] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < kKc; ++kk) {
            const float a = As[r][kk];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fmaf(Ws[g][u][kk], a, acc[g]);
        }
    }
    if (!live) return;
    const int node = p.nodes[m];
    float c, h;
    if constexpr (G == 3) {      // leaf: (i, o, u)
        const float zi = acc[0] + p.bias[j], zo = acc[1] + p.bias[H + j], zu = acc[2] + p.bias[2 * H + j];
        c = ptx::sigmoidf_(zi) * tanhf(zu);
        h = ptx::sigmoidf_(zo) * tanhf(c);
    } else {           // internal: (i, f_l, f_r, o, u)
        const float *cc = p.ccat + (int64_t)node * p.ldcat;
        const float zi = acc[0] + p.bias[j], zl = acc[1] + p.bias[H + j], zr = acc[2] + p.bias[2 * H + j];
        const float zo = acc[G > 3 ? 3 : 0] + p.bias[3 * H + j], zu = acc[G > 4 ? 4 : 0] + p.bias[4 * H + j];
        c = ptx::sigmoidf_(zi) * tanhf(zu) + ptx::sigmoidf_(zl) * cc[j] + ptx::sigmoidf_(zr) * cc[H + j];
        h = ptx::sigmoidf_(zo) * tanhf(c);
    }
    p.h_out[(int64_t)node * p.ldo + j] = h;
    p.c_out[(int64_t)node * p.ldo + j] = c;
    const int slot = p.parent_slot[m];
    if (slot >= 0) {
        const int64_t base = (int64_t)(slot >> 1) * p.ldcat + (slot & 1) * H + j;
        p.hcat[base] = h;
        p.ccat[base] = c;
    }
}

}  // namespace

cudaError_t launch_treelstm_level(const TreeParams &p, cudaStream_t s) {
    dim3 grid((p.H + kUnits - 1) / kUnits, (p.M + kNodes - 1) / kNodes);
    if (p.is_leaf) return launch_pdl(treelstm_level_kernel<3>, grid, dim3(kNodes * kUnits), 0, s, p);
    return launch_pdl(treelstm_level_kernel<5>, grid, dim3(kNodes * kUnits), 0, s, p);
}

}  // namespace nimble
