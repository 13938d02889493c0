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

// ---------------------------------------------------------------- whole forest, one launch
// The level loop runs on the device (the schedule — level offsets, node ids, input rows,
// parent slots — is device data), so a forest is ONE launch instead of one per level
// plus host round trips ("small kernels plus control flow").  Work item =
// one warp computing an 8-node x UPI-unit block of the level's Z for all G gates: lanes
// (unit = lane/KS, k-slice = lane%KS) stride K in float4s, the KS partial sums per unit are
// combined by a transpose-reduce that leaves one lane per node holding its G gate sums,
// which then applies the cell and writes h / c into the parent slot.
// Items are spread over every warp of a co-resident grid, so even a 3-node level keeps
// ~100 warps busy; a release/acquire counter barrier separates levels.
constexpr int kFThreads = 256;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFNodes = 8;       // nodes per warp item

// hcat / ccat rows written by the previous level: plain weak loads.  The level barrier's
// acquire fence invalidates L1 (and bar.sync orders the CTA behind it), so no stale line
// survives; __ldcg would compile to LDG.STRONG.GPU, which the compiler does not batch.
__device__ __forceinline__ float4 ld_cg4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float4 ld_nc4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

template <int G>
__device__ __forceinline__ void fma4(float (&acc)[G], const float4 (&w)[G], const float4 a) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
        acc[g] = fmaf(w[g].x, a.x, acc[g]);
        acc[g] = fmaf(w[g].y, a.y, acc[g]);
        acc[g] = fmaf(w[g].z, a.z, acc[g]);
        acc[g] = fmaf(w[g].w, a.w, acc[g]);
    }
}

// UPI hidden units per warp item, KS = 32 / UPI k-slice lanes per unit.  UPI = 4 reuses each
// A load across 4 units (throughput, big levels); UPI = 1 cuts the serial K steps per item
// from ceil(K/32) to ceil(K/128) (latency, small levels: each K step is one L2 round trip).
template <int G, bool LEAF, int UPI>
__device__ __forceinline__ void forest_level(const TreeForestParams &p, int beg, int end, int gw, int TW, int lane) {
    constexpr int KS = 32 / UPI;
    static_assert(KS >= 8, "the transpose-reduce needs >= 8 k-slice lanes per unit");
    const int H = p.H;
    const int K = LEAF ? p.I : 2 * H;
    const int K4 = K >> 2;
    const float *A = LEAF ? p.X : p.hcat;
    const int64_t lda = LEAF ? p.ldx : p.ldcat;
    const float *W = LEAF ? p.W_l : p.U;
    const float *bias = LEAF ? p.b_l : p.b_u;
    const int UG = (H + UPI - 1) / UPI;
    const int NT = (end - beg + kFNodes - 1) / kFNodes;
    const int items = NT * UG;
    const int ul = lane / KS, s = lane % KS;
    for (int item = gw; item < items; item += TW) {
        const int nt = item / UG, ug = item - nt * UG;
        const int j = ug * UPI + ul;
        const bool jv = j < H;
        const int jr = jv ? j : 0;
        // rows past the level end are clamped to the last node (their sums are discarded by
        // the cell's m < end test): no per-node branch, so all loads of a k step issue together.
        const float *arow[kFNodes];
#pragma unroll
        for (int r = 0; r < kFNodes; ++r) {
            const int m = min(beg + nt * kFNodes + r, end - 1);
            arow[r] = A + (int64_t)__ldg(p.rows + m) * lda;
        }
        float acc[kFNodes][G];
#pragma unroll
        for (int r = 0; r < kFNodes; ++r)
#pragma unroll
            for (int g = 0; g < G; ++g) acc[r][g] = 0.f;
        const float *wrow = W + (int64_t)jr * K;
        const int64_t gstride = (int64_t)H * K;
#pragma unroll 1
        for (int k4 = s; k4 < K4; k4 += KS) {
            float4 w[G], a[kFNodes];
#pragma unroll
            for (int g = 0; g < G; ++g) w[g] = ld_nc4(wrow + g * gstride + 4 * k4);
#pragma unroll
            for (int r = 0; r < kFNodes; ++r) a[r] = LEAF ? ld_nc4(arow[r] + 4 * k4) : ld_cg4(arow[r] + 4 * k4);
#pragma unroll
            for (int r = 0; r < kFNodes; ++r) fma4<G>(acc[r], w, a[r]);
        }
        // transpose-reduce over the KS k-slice lanes of each unit: three halving exchanges
        // (masks KS/2, KS/4, KS/8) split the 8 nodes over lane bits, then plain butterflies
        // finish the sum; lane s with s % (KS/8) == 0 holds node s / (KS/8).
        constexpr int M1 = KS / 2, M2 = KS / 4, M3 = KS / 8;
        float t4[4][G], t2[2][G], v[G];
        const bool b1 = s & M1, b2 = s & M2, b3 = s & M3;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float send = b1 ? acc[r][g] : acc[r + 4][g];
                const float keep = b1 ? acc[r + 4][g] : acc[r][g];
                t4[r][g] = keep + __shfl_xor_sync(0xffffffffu, send, M1);
            }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float send = b2 ? t4[r][g] : t4[r + 2][g];
                const float keep = b2 ? t4[r + 2][g] : t4[r][g];
                t2[r][g] = keep + __shfl_xor_sync(0xffffffffu, send, M2);
            }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float send = b3 ? t2[0][g] : t2[1][g];
            const float keep = b3 ? t2[1][g] : t2[0][g];
            v[g] = keep + __shfl_xor_sync(0xffffffffu, send, M3);
        }
#pragma unroll
        for (int mask = M3 / 2; mask >= 1; mask >>= 1)
#pragma unroll
            for (int g = 0; g < G; ++g) v[g] += __shfl_xor_sync(0xffffffffu, v[g], mask);
        if (s % M3) continue;
        const int m = beg + nt * kFNodes + s / M3;
        if (m >= end || !jv) continue;
        const int node = __ldg(p.nodes + m);
        float c, h;
        if constexpr (LEAF) {      // (i, o, u)
            const float zi = v[0] + bias[j], zo = v[1] + bias[H + j], zu = v[2] + bias[2 * H + j];
            c = ptx::sigmoidf_(zi) * tanhf(zu);
            h = ptx::sigmoidf_(zo) * tanhf(c);
        } else {                   // (i, f_l, f_r, o, u)
            const float *cc = p.ccat + (int64_t)node * p.ldcat;
            const float zi = v[0] + bias[j], zl = v[1] + bias[H + j], zr = v[2] + bias[2 * H + j];
            const float zo = v[G > 3 ? 3 : 0] + bias[3 * H + j], zu = v[G > 4 ? 4 : 0] + bias[4 * H + j];
            c = ptx::sigmoidf_(zi) * tanhf(zu) + ptx::sigmoidf_(zl) * cc[j] + ptx::sigmoidf_(zr) * cc[H + j];
            h = ptx::sigmoidf_(zo) * tanhf(c);
        }
        p.h_out[(int64_t)node * p.ldo + j] = h;
        p.c_out[(int64_t)node * p.ldo + j] = c;
        const int slot = __ldg(p.pslot + m);
        if (slot >= 0) {
            const int64_t base = (int64_t)(slot >> 1) * p.ldcat + (slot & 1) * H + j;
            p.hcat[base] = h;
            p.ccat[base] = c;
        }
    }
}

// Serial L2 round trips of a level for a UPI choice: item rounds x K steps per item.
__device__ __forceinline__ int level_steps(int n, int H, int K4, int TW, int upi) {
    const int items = (n + kFNodes - 1) / kFNodes * ((H + upi - 1) / upi);
    const int ks = 32 / upi;
    return (items + TW - 1) / TW * ((K4 + ks - 1) / ks);
}

// Poll with relaxed loads and take the acquire with ONE fence after the counter is seen:
// ld.acquire.gpu compiles to an L1 invalidate (CCTL.IVALL) per iteration, and a spinning
// CTA would keep wiping the L1 of the CTA computing next to it on the same SM.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kFThreads) treelstm_forest_kernel(const TreeForestParams p) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kFWarps + (threadIdx.x >> 5);
    const int TW = gridDim.x * kFWarps;
    for (int lv = 0; lv < p.n_levels; ++lv) {
        const int beg = __ldg(p.level_off + lv), end = __ldg(p.level_off + lv + 1);
        const int K4 = (lv == 0 ? p.I : 2 * p.H) >> 2;
        const bool wide = level_steps(end - beg, p.H, K4, TW, 4) <= level_steps(end - beg, p.H, K4, TW, 1);
        if (lv == 0) {
            if (wide) forest_level<3, true, 4>(p, beg, end, gw, TW, lane);
            else forest_level<3, true, 1>(p, beg, end, gw, TW, lane);
        } else {
            if (wide) forest_level<5, false, 4>(p, beg, end, gw, TW, lane);
            else forest_level<5, false, 1>(p, beg, end, gw, TW, lane);
        }
        if (p.trace && threadIdx.x == 0) p.trace[((size_t)blockIdx.x * 64 + (lv & 63)) * 2] = ptx::globaltimer();
        if (lv + 1 == p.n_levels) break;
        __syncthreads();
        if (threadIdx.x == 0) {     // level barrier: publish this CTA's h/c, wait for all CTAs
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p.counter), "r"(1u) : "memory");
            const unsigned target = (unsigned)(lv + 1) * gridDim.x;
            uint32_t spins = 0;
            while (ld_relaxed_u32(p.counter) < target) {
                __nanosleep(64);
                if (++spins == (1u << 26)) __trap();     // never hang the GPU on a protocol bug
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            if (p.trace) p.trace[((size_t)blockIdx.x * 64 + (lv & 63)) * 2 + 1] = ptx::globaltimer();
        }
        __syncthreads();
    }
}

}  // namespace

unsigned long long *lstm_trace_buffer();     // api.cu: the nimble_debug_trace buffer

cudaError_t launch_treelstm_forest(const TreeForestParams &p, cudaStream_t s) {
    static int occ = 0;
    if (occ == 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, treelstm_forest_kernel, kFThreads, 0);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
    }
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    const int64_t items = ((int64_t)p.max_level + kFNodes - 1) / kFNodes * p.H;   // 1-unit items
    int64_t grid = (items + kFWarps - 1) / kFWarps;
    grid = grid < (int64_t)sms * occ ? grid : (int64_t)sms * occ;
    if (grid < 1) grid = 1;
    e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    TreeForestParams q = p;
    q.trace = lstm_trace_buffer();
    void *args[] = {&q};
    return cudaLaunchCooperativeKernel((const void *)treelstm_forest_kernel, dim3((unsigned)grid), dim3(kFThreads),
                                       args, 0, s);
}

cudaError_t launch_treelstm_level(const TreeParams &p, cudaStream_t s) {
    dim3 grid((p.H + kUnits - 1) / kUnits, (p.M + kNodes - 1) / kNodes);
    if (p.is_leaf) return launch_pdl(treelstm_level_kernel<3>, grid, dim3(kNodes * kUnits), 0, s, p);
    return launch_pdl(treelstm_level_kernel<5>, grid, dim3(kNodes * kUnits), 0, s, p);
}

}  // namespace nimble
