// Two stacked LSTM layers over a runtime-length sequence as ONE persistent wavefront kernel
// (Nimble's LSTM LM; config 2 "2 layers, hidden 650", BJ:8).
//
// At global step s = 0..T, layer-1 CTAs compute h1_s (from the hoisted projection
// G1[s] = x_s W_ih1^T + b1 and W_hh1 h1_{s-1}) while layer-2 CTAs compute h2_{s-1} (from
// W_ih2 h1_{s-1} + W_hh2 h2_{s-2} + b2): both only need h1_{s-1}, so one synchronisation
// per step serves both layers -> T + 1 instead of 2T.  Every CTA keeps its gate rows of the
// weights resident in shared memory for the whole sequence; layer-2 CTAs own twice the rows
// (W_ih2 and W_hh2).  No separate grid barrier: h_t is published as tagged 64-bit words
// (t + 1, h) in parity ping-pong buffers and consumers poll the data itself (one L2 round
// trip per step).  Ping-pong safety: before a CTA overwrites slot t & 1 it has polled every
// CTA's later output (h1_{t-1} from layer 1, h2_{t-2} from layer 2), and each CTA produces
// those only after it consumed what the slot held.
#include <cstdlib>

#include "launch.h"
#include "ptx.cuh"

namespace nimble {

unsigned long long *lstm_trace_buffer();     // api.cu: the nimble_debug_trace buffer

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Lstm2Args {
    const float *G1; int64_t ldg;
    const float *Whh1, *Wih2, *Whh2; int64_t ldw;
    const float *b2;
    float *H1, *H2; int64_t ldh;
    float *hT, *cT;              // [2][H]
    unsigned long long *hbuf;    // [2 layers][2 ping-pong][H] tagged (t + 1) << 32 | float bits
    int T, H, n1, JB1, JB2;      // n1 layer-1 CTAs (JB1 units each), the rest layer 2 (JB2 units)
    unsigned long long *trace;   // debug: [2 CTAs][T+1 steps][4 stamps] or NULL
    // fused layer-1 input projection (X != NULL; register-resident variant only): G1[t] =
    // W_ih1 x_t + b1 is computed in the kernel from W_ih1 rows held in shared memory
    const float *X; int64_t ldx;
    const float *Wih1; int64_t ldwi;
    const float *b1;
    int I;
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int kMaxPer = 4;                      // H <= kMaxPer * blockDim (1024)
// read H tagged values of step `tag` into smem: all of this thread's words are requested
// at once (one L2 round trip), then only stale words are re-polled
__device__ __forceinline__ void gather_h(float *dst, const unsigned long long *src, int H, unsigned tag) {
    unsigned long long w[kMaxPer];
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) {
        const int k = threadIdx.x + i * blockDim.x;
        w[i] = (k < H) ? ld_relaxed_u64(src + k) : ((unsigned long long)tag << 32);
    }
    uint32_t spins = 0;
    for (;;) {
        bool done = true;
#pragma unroll
        for (int i = 0; i < kMaxPer; ++i) {
            if ((w[i] >> 32) != tag) {
                done = false;
                w[i] = ld_relaxed_u64(src + threadIdx.x + i * blockDim.x);
            }
        }
        if (done) break;
        if (++spins == (1u << 26)) __trap();           // never hang the GPU on a protocol bug
    }
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) {
        const int k = threadIdx.x + i * blockDim.x;
        if (k < H) dst[k] = __uint_as_float((unsigned)(w[i] & 0xffffffffu));
    }
}

constexpr int kRowsPerWarp = 8;                 // gate rows per matrix per CTA <= 8 * kWarps
// acc[rr] += W[row_rr] . x over the zero-padded row length Hp (multiple of 128): all of the
// warp's rows advance together, one independent FMA chain each, no per-element guards;
// 16-B shared-memory loads (a lane takes 4 consecutive k of every 128).
__device__ __forceinline__ void warp_rows_dot(float (&acc)[kRowsPerWarp], const float *W, const float *x, int Hp,
                                              int warp, int nrows, int lane) {
#pragma unroll 2
    for (int k = 4 * lane; k < Hp; k += 128) {
        const float4 xv = *reinterpret_cast<const float4 *>(x + k);
#pragma unroll
        for (int rr = 0; rr < kRowsPerWarp; ++rr) {
            const int r = warp + kWarps * rr;
            if (r < nrows) {
                const float4 wv = *reinterpret_cast<const float4 *>(W + (size_t)r * Hp + k);
                acc[rr] = fmaf(wv.x, xv.x, fmaf(wv.y, xv.y, fmaf(wv.z, xv.z, fmaf(wv.w, xv.w, acc[rr]))));
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads, 1) lstm2_kernel(const Lstm2Args a) {
    extern __shared__ float sm[];
    const int H = a.H;
    const bool l2 = (int)blockIdx.x >= a.n1;
    const int cta = l2 ? (int)blockIdx.x - a.n1 : (int)blockIdx.x;
    const int JB = l2 ? a.JB2 : a.JB1;
    const int j0 = cta * JB;
    const int R = 4 * JB;                       // gate rows per matrix
    const int nmat = l2 ? 2 : 1;
    const int Hp = 128 * ((H + 127) / 128);     // rows zero-padded to whole 128-wide warp chunks
    float *W = sm;                              // [nmat][R][Hp]
    float *x1 = W + (size_t)nmat * R * Hp;      // h1_{s-1} (zero-padded to Hp)
    float *x2 = x1 + Hp;                        // h2_{s-2} (layer 2 only)
    float *z = x2 + Hp;                         // [R]
    float *cs = z + R;                          // [JB]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // weights (static): staged before the grid-dependency wait, so with PDL this overlaps the
    // preceding input-projection GEMM.  One warp per row, lanes along k, asynchronous 8-byte
    // copies (cp.async, zero-filled past H): every copy of the CTA is in flight at once.
    const bool even = ((a.ldw & 1) == 0) && ((H & 1) == 0);
    for (int m = 0; m < nmat; ++m) {
        const float *src = l2 ? (m == 0 ? a.Wih2 : a.Whh2) : a.Whh1;
        for (int r = warp; r < R; r += kWarps) {
            const int g = r / JB, u = r - g * JB, j = j0 + u;
            const float *row = src + (int64_t)(g * H + (j < H ? j : 0)) * a.ldw;
            float *dst = W + ((size_t)m * R + r) * Hp;
            if (even) {
                for (int k = 2 * lane; k < Hp; k += 64) {
                    const uint32_t nbytes = (j < H && k < H) ? 8u : 0u;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(ptx::smem_u32(dst + k)),
                                 "l"(row + (k < H ? k : 0)), "r"(nbytes)
                                 : "memory");
                }
            } else {
                for (int k = lane; k < Hp; k += 32) dst[k] = (j < H && k < H) ? __ldg(row + k) : 0.f;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    for (int u = threadIdx.x; u < JB; u += kThreads) cs[u] = 0.f;
    for (int k = threadIdx.x; k < Hp; k += kThreads) { x1[k] = 0.f; x2[k] = 0.f; }
    __syncthreads();
    ptx::pdl_trigger();
    ptx::pdl_wait();                            // G1 (the input GEMM) and the workspace of the previous call

    unsigned long long *tr = nullptr;
    if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || (int)blockIdx.x == a.n1))
        tr = a.trace + (size_t)(blockIdx.x == 0 ? 0 : 1) * (a.T + 1) * 4;
    for (int s = 0; s <= a.T; ++s) {
        const int t = l2 ? s - 1 : s;           // the time step this CTA computes
        const bool active = t >= 0 && t < a.T;
        if (tr) tr[s * 4 + 0] = ptx::globaltimer();
        // layer 1: prefetch this step's hoisted input projection while the gather waits
        float gpre[4] = {0.f, 0.f, 0.f, 0.f};
        if (!l2 && active && threadIdx.x < JB && j0 + (int)threadIdx.x < H) {
            const float *g = a.G1 + (int64_t)t * a.ldg + j0 + threadIdx.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) gpre[q] = __ldg(g + q * H);
        }
        if (s > 0) {
            // h1_{s-1} (both layers), h2_{s-2} (layer 2): poll the tagged words themselves
            gather_h(x1, a.hbuf + (size_t)((s - 1) & 1) * H, H, (unsigned)s);
            // layer 2 gathers h2_{s-2}; layer 1 polls it too: every layer-2 CTA writes h2_{s-2}
            // only after consuming h1_{s-2}, so slot (s & 1) of h1 is free to overwrite
            if (s >= 2) gather_h(x2, a.hbuf + (size_t)(2 + ((s - 2) & 1)) * H, H, (unsigned)(s - 1));
            __syncthreads();
        }
        if (tr) tr[s * 4 + 1] = ptx::globaltimer();
        if (active) {
            float acc[kRowsPerWarp];
#pragma unroll
            for (int rr = 0; rr < kRowsPerWarp; ++rr) acc[rr] = 0.f;
            warp_rows_dot(acc, W, x1, Hp, warp, R, lane);
            if (l2) warp_rows_dot(acc, W + (size_t)R * Hp, x2, Hp, warp, R, lane);
#pragma unroll
            for (int rr = 0; rr < kRowsPerWarp; ++rr) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], o);
            }
            if (lane == 0) {
#pragma unroll
                for (int rr = 0; rr < kRowsPerWarp; ++rr)
                    if (warp + kWarps * rr < R) z[warp + kWarps * rr] = acc[rr];
            }
            __syncthreads();
            if (tr) tr[s * 4 + 2] = ptx::globaltimer();
            if (threadIdx.x < JB) {
                const int u = threadIdx.x, j = j0 + u;
                if (j < H) {
                    float zi, zf, zg, zo;
                    if (l2) {
                        zi = z[u] + a.b2[j]; zf = z[JB + u] + a.b2[H + j];
                        zg = z[2 * JB + u] + a.b2[2 * H + j]; zo = z[3 * JB + u] + a.b2[3 * H + j];
                    } else {
                        zi = z[u] + gpre[0]; zf = z[JB + u] + gpre[1]; zg = z[2 * JB + u] + gpre[2];
                        zo = z[3 * JB + u] + gpre[3];
                    }
                    const float c = ptx::sigmoidf_(zf) * cs[u] + ptx::sigmoidf_(zi) * tanhf(zg);
                    const float h = ptx::sigmoidf_(zo) * tanhf(c);
                    cs[u] = c;
                    st_relaxed_u64(a.hbuf + (size_t)((l2 ? 2 : 0) + (t & 1)) * H + j,
                                   ((unsigned long long)(t + 1) << 32) | __float_as_uint(h));
                    (l2 ? a.H2 : a.H1)[(int64_t)t * a.ldh + j] = h;
                    if (t == a.T - 1) {
                        a.hT[(l2 ? H : 0) + j] = h;
                        a.cT[(l2 ? H : 0) + j] = c;
                    }
                }
            }
        }
        __syncthreads();                        // z / x reuse in the next step
        if (tr) tr[s * 4 + 3] = ptx::globaltimer();
    }
    // leave the tagged buffers zeroed for the next call (no host memset on the hot path): the
    // last CTA to finish — every CTA has then consumed every word it polls — clears them
    __shared__ int is_last;
    unsigned *done = reinterpret_cast<unsigned *>(a.hbuf + 4 * (size_t)H);
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        for (int k = threadIdx.x; k < 4 * H; k += kThreads) a.hbuf[k] = 0ull;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *done = 0u;
    }
}

// ---- register-resident variant (H <= 672): 16 warps, each CTA's (matrix, gate-row) jobs
// spread over the warps (<= 4 per warp); a lane keeps k = lane + 32 i (i < NI) of each of its
// rows in registers for the whole sequence, so a step reads only x from shared memory (the
// shared-memory variant re-reads its whole weight block, ~170 KB, every step).
constexpr int kRegThreads = 512;
constexpr int kRegWarps = kRegThreads / 32;
constexpr int kJobsPerWarp = 4;

template <int NI, bool FUSE>
__global__ void __launch_bounds__(kRegThreads, 1) lstm2_reg_kernel(const Lstm2Args a) {
    extern __shared__ float sm[];
    const int H = a.H;
    const bool l2 = (int)blockIdx.x >= a.n1;
    const int cta = l2 ? (int)blockIdx.x - a.n1 : (int)blockIdx.x;
    const int JB = l2 ? a.JB2 : a.JB1;
    const int j0 = cta * JB;
    const int R = 4 * JB;                       // gate rows per matrix
    const int nmat = l2 ? 2 : 1;
    const int J = nmat * R;                     // jobs: (matrix, row)
    constexpr int Hp = 32 * NI;
    float *x1 = sm;                             // h1_{s-1} (zero-padded to Hp)
    float *x2 = x1 + Hp;                        // h2_{s-2} (layer 2 only)
    float *z = x2 + Hp;                         // [2][R] per-matrix gate pre-activations
    float *cs = z + 2 * R;                      // [JB]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // fused input projection (layer-1 CTAs): W_ih1 rows [R][Ip], x_t [Ip], gin [R]
    const bool fuse = FUSE && !l2;              // compile-time: the unfused kernel carries none of it
    const int Ip = 32 * ((a.I + 31) / 32);
    float *xin = cs + 4 * ((JB + 3) / 4);       // 16-B aligned
    float *gin = xin + Ip;
    float *Wi = gin + 4 * ((R + 3) / 4);
    if (fuse) {
        // rows of W_ih1 -> shared memory (static weights: before the grid-dependency wait), 4-B
        // cp.async, zero-filled past I and for units past H
        for (int r = warp; r < R; r += kRegWarps) {
            const int g = r / JB, u = r - g * JB, j = j0 + u;
            const float *row = a.Wih1 + (int64_t)(g * H + (j < H ? j : 0)) * a.ldwi;
            for (int k = lane; k < Ip; k += 32) {
                const uint32_t nbytes = (j < H && k < a.I) ? 4u : 0u;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(ptx::smem_u32(Wi + (size_t)r * Ip + k)),
                             "l"(row + (k < a.I ? k : 0)), "r"(nbytes)
                             : "memory");
            }
        }
    }

    // weights -> registers (static: before the grid-dependency wait, overlapping the input GEMM)
    float w[kJobsPerWarp][NI];
    int jm[kJobsPerWarp];                       // matrix of job q (-1: none)
#pragma unroll
    for (int q = 0; q < kJobsPerWarp; ++q) {
        const int jb = warp + kRegWarps * q;
        jm[q] = jb < J ? jb / R : -1;
        const int r = jb < J ? jb % R : 0;
        const int g = r / JB, u = r - g * JB, j = j0 + u;
        const float *src = l2 ? (jm[q] == 0 ? a.Wih2 : a.Whh2) : a.Whh1;
        const float *row = src + (int64_t)(g * H + (j < H ? j : 0)) * a.ldw;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int k = lane + 32 * i;
            w[q][i] = (jm[q] >= 0 && j < H && k < H) ? __ldg(row + k) : 0.f;
        }
    }
    for (int u = threadIdx.x; u < JB; u += kRegThreads) cs[u] = 0.f;
    for (int k = threadIdx.x; k < Hp; k += kRegThreads) { x1[k] = 0.f; x2[k] = 0.f; }
    if (fuse) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    ptx::pdl_trigger();
    ptx::pdl_wait();                            // G1 / X and the workspace of the previous call

    unsigned long long *tr = nullptr;
    if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || (int)blockIdx.x == a.n1))
        tr = a.trace + (size_t)(blockIdx.x == 0 ? 0 : 1) * (a.T + 1) * 4;
    // fused input projection: x_t is prefetched into registers one step ahead (its global load
    // latency never sits on a step), two values per thread (Ip <= 2 * kRegThreads)
    float xr0 = 0.f, xr1 = 0.f;
    if (fuse) {
        const int k0 = threadIdx.x, k1 = threadIdx.x + kRegThreads;
        xr0 = k0 < a.I ? __ldg(a.X + k0) : 0.f;
        xr1 = k1 < a.I ? __ldg(a.X + k1) : 0.f;
    }
    for (int s = 0; s <= a.T; ++s) {
        const int t = l2 ? s - 1 : s;           // the time step this CTA computes
        const bool active = t >= 0 && t < a.T;
        if (tr) tr[s * 4 + 0] = ptx::globaltimer();
        float gpre[4] = {0.f, 0.f, 0.f, 0.f};
        if (fuse && active) {
            // W_ih1 x_t for this CTA's gate rows while the other CTAs' h_{t-1} is in flight: it
            // needs no h, so it sits before the gather (off the step's critical path)
            if (threadIdx.x < Ip) xin[threadIdx.x] = xr0;
            if (threadIdx.x + kRegThreads < Ip) xin[threadIdx.x + kRegThreads] = xr1;
            if (t + 1 < a.T) {                  // prefetch x_{t+1}
                const int k0 = threadIdx.x, k1 = threadIdx.x + kRegThreads;
                xr0 = k0 < a.I ? __ldg(a.X + (int64_t)(t + 1) * a.ldx + k0) : 0.f;
                xr1 = k1 < a.I ? __ldg(a.X + (int64_t)(t + 1) * a.ldx + k1) : 0.f;
            }
            __syncthreads();
            // a warp's (<= 4) rows advance together: independent FMA chains, one reduction pass
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            for (int k = lane; k < Ip; k += 32) {
                const float xv = xin[k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = warp + kRegWarps * q;
                    if (r < R) acc[q] = fmaf(Wi[(size_t)r * Ip + k], xv, acc[q]);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (warp + kRegWarps * q < R) gin[warp + kRegWarps * q] = acc[q];
            }
            __syncthreads();
            if (threadIdx.x < JB && j0 + (int)threadIdx.x < H) {
                const int u = threadIdx.x, j = j0 + u;
#pragma unroll
                for (int q = 0; q < 4; ++q) gpre[q] = gin[q * JB + u] + __ldg(a.b1 + q * H + j);
            }
        } else if (!l2 && active && threadIdx.x < JB && j0 + (int)threadIdx.x < H) {
            const float *g = a.G1 + (int64_t)t * a.ldg + j0 + threadIdx.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) gpre[q] = __ldg(g + q * H);
        }
        if (s > 0) {
            gather_h(x1, a.hbuf + (size_t)((s - 1) & 1) * H, H, (unsigned)s);
            if (s >= 2) gather_h(x2, a.hbuf + (size_t)(2 + ((s - 2) & 1)) * H, H, (unsigned)(s - 1));
            __syncthreads();
        }
        if (tr) tr[s * 4 + 1] = ptx::globaltimer();
        if (active) {
            float acc[kJobsPerWarp];
#pragma unroll
            for (int q = 0; q < kJobsPerWarp; ++q) acc[q] = 0.f;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const float xa = x1[lane + 32 * i];
                const float xb = l2 ? x2[lane + 32 * i] : 0.f;
#pragma unroll
                for (int q = 0; q < kJobsPerWarp; ++q) acc[q] = fmaf(w[q][i], jm[q] == 1 ? xb : xa, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < kJobsPerWarp; ++q) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            }
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < kJobsPerWarp; ++q) {
                    const int jb = warp + kRegWarps * q;
                    if (jb < J) z[jb] = acc[q];          // z[m R + r]
                }
            }
            __syncthreads();
            if (tr) tr[s * 4 + 2] = ptx::globaltimer();
            if (threadIdx.x < JB) {
                const int u = threadIdx.x, j = j0 + u;
                if (j < H) {
                    float zi, zf, zg, zo;
                    if (l2) {
                        zi = z[u] + z[R + u] + a.b2[j];
                        zf = z[JB + u] + z[R + JB + u] + a.b2[H + j];
                        zg = z[2 * JB + u] + z[R + 2 * JB + u] + a.b2[2 * H + j];
                        zo = z[3 * JB + u] + z[R + 3 * JB + u] + a.b2[3 * H + j];
                    } else {
                        zi = z[u] + gpre[0]; zf = z[JB + u] + gpre[1]; zg = z[2 * JB + u] + gpre[2];
                        zo = z[3 * JB + u] + gpre[3];
                    }
                    const float c = ptx::sigmoidf_(zf) * cs[u] + ptx::sigmoidf_(zi) * tanhf(zg);
                    const float h = ptx::sigmoidf_(zo) * tanhf(c);
                    cs[u] = c;
                    st_relaxed_u64(a.hbuf + (size_t)((l2 ? 2 : 0) + (t & 1)) * H + j,
                                   ((unsigned long long)(t + 1) << 32) | __float_as_uint(h));
                    (l2 ? a.H2 : a.H1)[(int64_t)t * a.ldh + j] = h;
                    if (t == a.T - 1) {
                        a.hT[(l2 ? H : 0) + j] = h;
                        a.cT[(l2 ? H : 0) + j] = c;
                    }
                }
            }
        }
        __syncthreads();                        // z / x reuse in the next step
        if (tr) tr[s * 4 + 3] = ptx::globaltimer();
    }
    __shared__ int is_last;
    unsigned *done = reinterpret_cast<unsigned *>(a.hbuf + 4 * (size_t)H);
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        for (int k = threadIdx.x; k < 4 * H; k += kRegThreads) a.hbuf[k] = 0ull;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *done = 0u;
    }
}

template <int NI, bool FUSE>
cudaError_t launch_reg_t(const Lstm2Args &a, unsigned grid, cudaStream_t s) {
    const int JBm = a.JB1 > a.JB2 ? a.JB1 : a.JB2;
    size_t smem = sizeof(float) * ((size_t)2 * 32 * NI + 2 * 4 * JBm + JBm + 64);
    if (a.X) {                                  // + x_t, gin, W_ih1 rows of a layer-1 CTA
        const size_t Ip = 32 * (((size_t)a.I + 31) / 32);
        smem += sizeof(float) * (Ip + 4 * a.JB1 + 8 + (size_t)4 * a.JB1 * Ip);
        static size_t attr = 0;
        if (attr < smem) {
            cudaError_t e = cudaFuncSetAttribute(lstm2_reg_kernel<NI, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            attr = smem;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRegThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, lstm2_reg_kernel<NI, FUSE>, a);
}
template <int NI>
cudaError_t launch_reg(const Lstm2Args &a, unsigned grid, cudaStream_t s) {
    return a.X ? launch_reg_t<NI, true>(a, grid, s) : launch_reg_t<NI, false>(a, grid, s);
}

}  // namespace

size_t lstm2_workspace_bytes(int64_t H) { return sizeof(unsigned long long) * (4 * (size_t)H + 2); }   // + exit counter

cudaError_t launch_lstm2_seq(const float *G1, int64_t ldg, const float *Whh1, const float *Wih2, const float *Whh2,
                             int64_t ldw, const float *b2, float *H1, float *H2, int64_t ldh, float *hT, float *cT,
                             int64_t T, int64_t H, void *workspace, cudaStream_t s, const Lstm2Input *fused) {
    // 3 : 1 split of the SMs (layer-2 CTAs own two matrices), <= 148 co-resident CTAs
    int n1 = 48;
    const int JB1 = (int)((H + n1 - 1) / n1);
    n1 = (int)((H + JB1 - 1) / JB1);
    int n2 = 2 * n1;
    const int JB2 = (int)((H + n2 - 1) / n2);
    n2 = (int)((H + JB2 - 1) / JB2);
    const int64_t Hp = 128 * ((H + 127) / 128);
    const size_t smem1 = sizeof(float) * ((size_t)4 * JB1 * Hp + 2 * Hp + 4 * JB1 + JB1);
    const size_t smem2 = sizeof(float) * ((size_t)8 * JB2 * Hp + 2 * Hp + 4 * JB2 + JB2);
    const size_t smem = smem1 > smem2 ? smem1 : smem2;
    if (smem > 232448 - 1024 || n1 + n2 > 148 || 4 * JB1 > 8 * kWarps || 4 * JB2 > 8 * kWarps) return cudaErrorInvalidValue;
    static size_t attr = 0;                    // the kernel also has a few bytes of static smem
    if (attr < smem) {
        cudaError_t e = cudaFuncSetAttribute(lstm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    Lstm2Args a;
    a.G1 = G1; a.ldg = ldg; a.Whh1 = Whh1; a.Wih2 = Wih2; a.Whh2 = Whh2; a.ldw = ldw; a.b2 = b2;
    a.H1 = H1; a.H2 = H2; a.ldh = ldh; a.hT = hT; a.cT = cT;
    a.hbuf = static_cast<unsigned long long *>(workspace);
    a.T = (int)T; a.H = (int)H; a.n1 = n1; a.JB1 = JB1; a.JB2 = JB2;
    a.trace = lstm_trace_buffer();
    a.X = nullptr; a.ldx = 0; a.Wih1 = nullptr; a.ldwi = 0; a.b1 = nullptr; a.I = 0;
    if (fused) {
        a.X = fused->X; a.ldx = fused->ldx; a.Wih1 = fused->Wih1; a.ldwi = fused->ldwi; a.b1 = fused->b1;
        a.I = (int)fused->I;
    }
    // register-resident weights when every CTA's (matrix, row) jobs fit 4 per warp and a row's
    // k-slice per lane fits NI <= 21 registers (H <= 672: config 2's 650, the paper's 512)
    static const bool reg_on = [] { const char *e = std::getenv("NIMBLE_LSTM_REG"); return !(e && e[0] == '0'); }();
    const int ni = (int)((H + 31) / 32);
    const bool fuse_fits = !fused || sizeof(float) * (32 * ((fused->I + 31) / 32) * (4 * (size_t)JB1 + 1) + 4 * JB1) +
                                         sizeof(float) * ((size_t)2 * 32 * ni + 12 * JB1 + 64) <= 232448 - 1024;
    const bool fuse_shape = !fused || (32 * ((fused->I + 31) / 32) <= 2 * kRegThreads && 4 * JB1 <= 4 * kRegWarps);
    if (fused && !(reg_on && ni <= 21 && fuse_fits && fuse_shape)) return cudaErrorNotSupported;   // caller composes GEMM + kernel
    if (reg_on && ni <= 21 && 4 * JB1 <= kRegWarps * kJobsPerWarp && 8 * JB2 <= kRegWarps * kJobsPerWarp) {
        const unsigned grid = (unsigned)(n1 + n2);
        if (ni <= 8) return launch_reg<8>(a, grid, s);
        if (ni <= 12) return launch_reg<12>(a, grid, s);
        if (ni <= 16) return launch_reg<16>(a, grid, s);
        return launch_reg<21>(a, grid, s);
    }
    // the workspace is zero on entry (caller-zeroed before the first call; every call leaves it
    // zeroed): tag 0 = not yet written.  Cooperative (all CTAs co-resident: they poll each other)
    // and programmatic (the weight staging overlaps the preceding kernel).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n1 + n2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, lstm2_kernel, a);
}

}  // namespace nimble
