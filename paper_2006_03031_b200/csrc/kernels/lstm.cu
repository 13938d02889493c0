// Fused dynamic-length LSTM layer (Nimble's LSTM benchmark, PAPER.md:575-576,
// PAPER.md:593-597): the VM's for-loop control flow becomes a device loop over the
// runtime T inside ONE persistent cooperative kernel.  Each CTA owns a slice of
// hidden units and keeps the matching 4 gate rows of W_hh resident in shared memory
// for the whole sequence; per step it reads h_{t-1} (L2), computes its W_hh h
// rows, adds the hoisted input projection G[t] = x_t W_ih^T + b (one dense_dyn
// over all T), applies the gates and writes h_t; a grid-wide
// barrier (one release/acquire counter) separates steps.
#include <cooperative_groups.h>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSmem = 200 * 1024;

struct LstmArgs {
    const float *G; int64_t ldg;
    const float *W; int64_t ldw;
    const float *h0, *c0;
    float *Hs; int64_t ldh;
    float *hT, *cT;
    float *hbuf;            // [2][H] ping-pong h broadcast buffer
    unsigned *counter;      // grid barrier counter (zeroed before launch)
    int T, H, JB;           // JB hidden units per CTA
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kThreads, 1) lstm_seq_kernel(const LstmArgs a) {
    extern __shared__ float sm[];
    const int H = a.H, JB = a.JB, R = 4 * JB;
    float *Ws = sm;                       // [R][H]   row g*JB+u = W_hh[g*H + j0 + u]
    float *hs = Ws + (size_t)R * H;       // [H]      h_{t-1}
    float *zs = hs + H;                   // [R]      W_hh h_{t-1} for this CTA's rows
    float *cs = zs + R;                   // [JB]     cell state of owned units
    const int j0 = blockIdx.x * JB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned nct = gridDim.x;

    for (int e = threadIdx.x; e < R * H; e += kThreads) {
        const int r = e / H, k = e % H;
        const int g = r / JB, u = r % JB;
        const int j = j0 + u;
        Ws[e] = (j < H) ? a.W[(int64_t)(g * H + j) * a.ldw + k] : 0.f;
    }
    for (int u = threadIdx.x; u < JB; u += kThreads) {
        const int j = j0 + u;
        cs[u] = (j < H && a.c0) ? a.c0[j] : 0.f;
    }
    for (int k = threadIdx.x; k < H; k += kThreads) hs[k] = a.h0 ? a.h0[k] : 0.f;
    __syncthreads();

    for (int t = 0; t < a.T; ++t) {
        if (t > 0) {
            const float *src = a.hbuf + (size_t)(t & 1) * H;
            for (int k = threadIdx.x; k < H; k += kThreads) hs[k] = __ldcg(src + k);   // L2, not stale L1
            __syncthreads();
        }
        for (int r = warp; r < R; r += kWarps) {
            const float *w = Ws + (size_t)r * H;
            float acc = 0.f;
            for (int k = lane; k < H; k += 32) acc = fmaf(w[k], hs[k], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) zs[r] = acc;
        }
        __syncthreads();
        if (threadIdx.x < JB) {
            const int u = threadIdx.x, j = j0 + u;
            if (j < H) {
                const float *g = a.G + (int64_t)t * a.ldg;
                const float zi = zs[0 * JB + u] + g[j];
                const float zf = zs[1 * JB + u] + g[H + j];
                const float zg = zs[2 * JB + u] + g[2 * H + j];
                const float zo = zs[3 * JB + u] + g[3 * H + j];
                const float c = ptx::sigmoidf_(zf) * cs[u] + ptx::sigmoidf_(zi) * tanhf(zg);
                const float h = ptx::sigmoidf_(zo) * tanhf(c);
                cs[u] = c;
                a.hbuf[(size_t)((t + 1) & 1) * H + j] = h;
                a.Hs[(int64_t)t * a.ldh + j] = h;
                if (t == a.T - 1) { a.hT[j] = h; a.cT[j] = c; }
            }
        }
        if (t + 1 < a.T) {
            // grid barrier: release our h slice, wait for every CTA's
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.counter), "r"(1u) : "memory");
                const unsigned target = (unsigned)(t + 1) * nct;
                uint32_t spins = 0;
                while (ld_acquire(a.counter) < target) {
                    if (++spins == (1u << 28)) __trap();     // never hang the GPU on a protocol bug
                }
            }
            __syncthreads();
        }
    }
}

int units_per_cta(int64_t H) { return (int)((H + 127) / 128); }

size_t lstm_smem(int64_t H, int JB) { return sizeof(float) * ((size_t)4 * JB * H + H + 4 * JB + JB); }

}  // namespace

size_t lstm_workspace_bytes(int64_t H) { return sizeof(float) * 2 * (size_t)H + 256; }

cudaError_t launch_lstm_seq(const float *G, int64_t ldg, const float *W_hh, int64_t ldw, const float *h0,
                            const float *c0, float *H_seq, int64_t ldh, float *hT, float *cT, int64_t T, int64_t H,
                            void *workspace, cudaStream_t s) {
    const int JB = units_per_cta(H);
    const size_t smem = lstm_smem(H, JB);
    if (smem > (size_t)kMaxSmem) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(lstm_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    LstmArgs a;
    a.G = G; a.ldg = ldg; a.W = W_hh; a.ldw = ldw; a.h0 = h0; a.c0 = c0;
    a.Hs = H_seq; a.ldh = ldh; a.hT = hT; a.cT = cT;
    a.hbuf = static_cast<float *>(workspace);
    a.counter = reinterpret_cast<unsigned *>(static_cast<char *>(workspace) + sizeof(float) * 2 * (size_t)H);
    a.T = (int)T; a.H = (int)H; a.JB = JB;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    const unsigned nct = (unsigned)((H + JB - 1) / JB);
    void *args[] = {&a};
    return cudaLaunchCooperativeKernel((const void *)lstm_seq_kernel, dim3(nct), dim3(kThreads), args, smem, s);
}

}  // namespace nimble
