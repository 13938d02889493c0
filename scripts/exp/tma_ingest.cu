// Experiment: per-SM TMA ingest rate (bytes/clk) as a function of bytes in flight, box shape,
// cluster multicast and grid size.  No MMA: a producer thread keeps `stages` 16-KB-class
// boxes in flight into a smem ring; a consumer thread releases each stage as soon as it lands
// (with multicast: to every CTA of the cluster).  Answers: is the GEMM main loop (~50 B/clk per
// SM measured) bound by latency x bytes-in-flight, by a per-SM request rate, or by L2?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ingest tma_ingest.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void expect_tx_relaxed(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ int g_wait_mode;   // 0 try_wait (no hint), 1 test_wait spin, 2 try_wait with a 0-ns suspend hint
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
    const int mode = g_wait_mode;
    if (mode == 1) {
        asm volatile("{\n.reg .pred p;\nW1: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(su32(b)), "r"(par) : "memory");
    } else if (mode == 2) {
        asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n@!p bra W2;\n}" ::"r"(su32(b)), "r"(par), "r"(0) : "memory");
    } else {
        asm volatile("{\n.reg .pred p;\nW0: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W0;\n}" ::"r"(su32(b)), "r"(par) : "memory");
    }
}
__device__ __forceinline__ void arrive_remote(uint64_t *b, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(b)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void load2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void load2d_mc(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, uint16_t mask) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "h"(mask) : "memory");
}

struct P {
    int stages, iters, csize, rows_per_cta_box, boxes_per_stage, row_span, col_blocks;
    unsigned long long *out;   // per CTA: clk
    int kdepth;                // 3-D box: kdepth consecutive 64-column blocks per box
    int bulk1d;                // 1: plain cp.async.bulk of box_bytes contiguous bytes instead of tensor boxes
    const uint8_t *gbase;
    int same_box;              // 1: every load reads the CTA's first box (pure L2-hit stream)
    int nsplit;                // variant 7: producer warps sharing each stage
    int variant;               // 0 plain, 1 prefetch.tensormap, 2 map in global memory, 3 two producer threads,
                               // 4 prefetch + no "memory" clobber loads
    const CUtensorMap *gmap;   // variant 2
    long long *ts;             // CTA 0: [it] issue clk, [4096 + it] complete clk
};
__device__ __forceinline__ void load3d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// stage = boxes_per_stage boxes of {64 cols, rows_per_cta_box * csize rows}; with multicast each
// CTA of a cluster loads rows_per_cta_box rows of every box and multicasts them to all.
__global__ void __launch_bounds__(288) ingest(const __grid_constant__ CUtensorMap tm, P p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
    const int box_rows = p.rows_per_cta_box * p.csize;
    const int box_bytes = box_rows * 128 * p.kdepth;
    const int stage_bytes = box_bytes * p.boxes_per_stage;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + p.stages * stage_bytes);
    uint64_t *empty = full + p.stages;
    const uint32_t rank = p.csize > 1 ? ctarank() : 0;
    const CUtensorMap *mp = p.variant == 2 ? p.gmap : &tm;
    if ((p.variant == 1 || p.variant >= 3) && (threadIdx.x == 0 || threadIdx.x == 64))
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)mp) : "memory");
    if (p.variant == 2 && threadIdx.x == 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)mp) : "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) { bar_init(&full[s], p.variant == 7 ? p.nsplit : 1); bar_init(&empty[s], p.csize * (p.variant == 7 ? p.nsplit : 1)); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (p.csize > 1) cluster_sync();
    const int cluster_id = blockIdx.x / p.csize;
    const int row0 = (cluster_id * box_rows * p.boxes_per_stage) % p.row_span;
    long long t0 = clock64();
    const int nprod = p.variant == 3 ? 2 : 1;
    const int pid = threadIdx.x == 0 ? 0 : (threadIdx.x == 64 ? 1 : -1);
    const int wsp = (threadIdx.x & 31) == 0 ? (int)(threadIdx.x >> 5) : -1;     // variant 7: warp id of lane 0
    if (p.variant == 7 && wsp >= 1 && wsp <= p.nsplit) {
        const int w = wsp - 1;
        int s = 0; uint32_t ph = 0;
        const int nb = (p.boxes_per_stage - w + p.nsplit - 1) / p.nsplit;   // boxes this warp issues per stage
        for (int it = 0; it < p.iters; ++it) {
            if (it >= p.stages) wait(&empty[s], ph ^ 1);
            expect_tx(&full[s], nb * box_bytes);
            const int cb = it % p.col_blocks;
            for (int b = w; b < p.boxes_per_stage; b += p.nsplit) {
                uint8_t *dst = sm + s * stage_bytes + b * box_bytes;
                load2d(dst, mp, &full[s], cb * 64, row0 + b * box_rows);
            }
            if (++s == p.stages) { s = 0; ph ^= 1; }
        }
    } else if (p.variant == 7) {
        if (threadIdx.x == 0) {     // consumer
            int s = 0; uint32_t ph = 0;
            for (int it = 0; it < p.iters; ++it) {
                wait(&full[s], ph);
                if (blockIdx.x == 0 && it < 4096) p.ts[4096 + it] = clock64();
                for (int c = 0; c < p.nsplit; ++c) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
                if (++s == p.stages) { s = 0; ph ^= 1; }
            }
            p.out[blockIdx.x] = clock64() - t0;
        }
    } else if (pid >= 0 && pid < nprod) {
        int s = pid; uint32_t ph = 0;
        for (int it = pid; it < p.iters; it += nprod) {
            if (it >= p.stages) wait(&empty[s], ph ^ 1);
            if (p.variant == 4) {
                if (it == 0) for (int q = 0; q < p.stages; ++q) expect_tx(&full[q], stage_bytes);
                else if (it >= p.stages) expect_tx(&full[s], stage_bytes);
            } else if (p.variant == 6) {
                expect_tx_relaxed(&full[s], stage_bytes);
            } else {
                expect_tx(&full[s], stage_bytes);
            }
            const int cb = p.same_box ? 0 : it % p.col_blocks;
            if (blockIdx.x == 0 && it < 4096 && p.variant != 5) p.ts[it] = clock64();
            for (int b = 0; b < p.boxes_per_stage; ++b) {
                uint8_t *dst = sm + s * stage_bytes + b * box_bytes + rank * p.rows_per_cta_box * 128;
                const int r = row0 + b * box_rows + rank * p.rows_per_cta_box;
                if (p.bulk1d) bulk1d(dst, p.gbase + ((size_t)r * 2048 + (size_t)cb * box_bytes) % ((size_t)p.row_span * 2048), box_bytes, &full[s]);
                else if (p.kdepth > 1) load3d(dst, &tm, &full[s], 0, r, (cb * p.kdepth) % p.col_blocks);
                else if (p.csize > 1) load2d_mc(dst, mp, &full[s], cb * 64, r, (uint16_t)((1u << p.csize) - 1));
                else load2d(dst, mp, &full[s], cb * 64, r);
            }
            s += nprod;
            if (s >= p.stages) { s -= p.stages; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < p.iters; ++it) {
            wait(&full[s], ph);
            if (blockIdx.x == 0 && it < 4096) p.ts[4096 + it] = clock64();
            for (int c = 0; c < p.csize; ++c) {
                if (p.csize > 1) arrive_remote(&empty[s], c);
                else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
            if (++s == p.stages) { s = 0; ph ^= 1; }
        }
        p.out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (p.csize > 1) cluster_sync();
}

int main(int argc, char **argv) {
    const int rows = 32768, cols = 1024;          // 64 MB bf16: fits L2 (126 MB), hot after the first pass
    void *buf;
    CK(cudaMalloc(&buf, (size_t)rows * cols * 2));
    CK(cudaMemset(buf, 1, (size_t)rows * cols * 2));
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    unsigned long long *out;
    CK(cudaMalloc(&out, 4096 * 8));
    long long *ts;
    CK(cudaMalloc(&ts, 8192 * 8));
    CUtensorMap *gm;
    CK(cudaMalloc(&gm, sizeof(CUtensorMap)));
    CK(cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    printf("same grid csize box_rows kdepth bulk1d boxes/stage stage_KB stages inflight_KB | B/clk/CTA(med) GB/s/CTA  aggregate_TB/s  us\n");
    struct Cfg { int grid, csize, rpcb, bps, stages, kd, b1d, same, var, nsplit; };
    std::vector<Cfg> cfgs;
    cfgs.push_back({148, 1, 128, 2, 6, 1, 0, 0, 0, 1});
    for (int ns : {1, 2, 4}) cfgs.push_back({148, 1, 128, 4, 3, 1, 0, 0, 7, ns});     // 64 KB stages, 4 boxes of 16 KB
    for (int ns : {2}) cfgs.push_back({148, 1, 128, 2, 6, 1, 0, 0, 7, ns});            // 32 KB stages (A + B)
    for (int ns : {4, 8}) cfgs.push_back({148, 1, 64, 8, 3, 1, 0, 0, 7, ns});         // 64 KB stages, 8 boxes of 8 KB
    for (int ns : {2, 4}) cfgs.push_back({8, 1, 128, 4, 3, 1, 0, 0, 7, ns});
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    CK(cudaMemcpyToSymbol(g_wait_mode, &mode, sizeof(int)));
    printf("wait mode %d (0 try_wait, 1 test_wait spin, 2 try_wait hint 0)\n", mode);
    for (auto c : cfgs) {
        const int box_rows = c.rpcb * c.csize;
        CUtensorMap tm;
        CUresult r;
        if (c.kd > 1) {        // {64 k, rows, k-blocks}: strides row = cols*2, k-block = 128 B
            cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
            cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
            cuuint32_t box[3] = {64, (cuuint32_t)c.rpcb, (cuuint32_t)c.kd}, es[3] = {1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
            cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)c.rpcb}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        P p{c.stages, 2048, c.csize, c.rpcb, c.bps, rows - box_rows * c.bps, cols / 64, out, c.kd, c.b1d,
            (const uint8_t *)buf, c.same, c.nsplit, c.var, gm, ts};
        CK(cudaMemcpy(gm, &tm, sizeof(tm), cudaMemcpyHostToDevice));
        const int stage_bytes = box_rows * 128 * c.bps * c.kd;
        const size_t smem = 1024 + (size_t)c.stages * stage_bytes + 256;
        if (smem > 232448) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(288);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) CK(cudaLaunchKernelEx(&cfg, ingest, tm, p));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, ingest, tm, p));
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> h(c.grid);
        CK(cudaMemcpy(h.data(), out, 8 * c.grid, cudaMemcpyDeviceToHost));
        std::vector<unsigned long long> s(h);
        std::sort(s.begin(), s.end());
        const double med = (double)s[s.size() / 2];
        const double bytes_per_cta = (double)p.iters * stage_bytes;          // bytes landing in each CTA's smem
        const double bpc = bytes_per_cta / med;
        const double agg_req = (double)c.grid * p.iters * stage_bytes / c.csize / (ms * 1e-3) / 1e12;   // L2 bytes read
        std::vector<long long> t(8192);
        CK(cudaMemcpy(t.data(), ts, 8192 * 8, cudaMemcpyDeviceToHost));
        std::vector<long long> lat;
        for (int i = 100; i < 400; ++i) lat.push_back(t[4096 + i] - t[i]);
        std::sort(lat.begin(), lat.end());
        const double per = (double)(t[4096 + 400] - t[4096 + 100]) / 300.0;
        printf("  first issues:");
        for (int i = 0; i < 12; ++i) printf(" %lld", t[i] - t[0]);
        printf("\n  completes:   ");
        for (int i = 0; i < 12; ++i) printf(" %lld", t[4096 + i] - t[0]);
        printf("\n");
        printf("  [CTA0 stage issue->complete clk: med %lld p90 %lld; complete->complete %.0f; => in flight ~%.1f]\n",
               lat[lat.size() / 2], lat[lat.size() * 9 / 10], per, lat[lat.size() / 2] / per);
        printf("var %d nsplit %d: ", c.var, c.nsplit);
        printf("%4d %4d %5d %8d %6d %6d %11d %8d %6d %11d | %12.1f %8.1f %14.2f %8.1f\n", c.same, c.grid, c.csize, box_rows, c.kd, c.b1d, c.bps,
               stage_bytes / 1024, c.stages, c.stages * stage_bytes / 1024, bpc, bpc * clk_khz * 1e3 / 1e9, agg_req,
               ms * 1e3);
    }
    return 0;
}
