// Experiment: steady-state per-SM TMA ingest (bytes/clk) of a GEMM-like smem ring, with no
// stores on the producer path (tma_ingest.cu's per-stage timestamp store perturbed it).
// 148 CTAs (one per SM); a ring of `stages` stages of `boxes` boxes; producer warps issue the
// boxes of each stage (box b by warp b % nprod), a consumer thread waits for a stage and
// releases it at once.  Data: 64 MB bf16, L2-resident after the first pass; each CTA streams
// its own rows (like the A / B tiles of a GEMM, which are L2 hits for most CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW0: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W0;\n}" ::"r"(su32(b)), "r"(par) : "memory");
}

struct P {
    int stages, boxes, nprod, iters, box_rows, kd, rows_total, kblocks;
    long long *out;
    int csize;           // > 1: cluster of csize CTAs; box b is issued by rank b % csize, multicast to all
    int mode;            // 0 tensor / try_wait, 1 consumer test_wait spin, 2 1-D cp.async.bulk, 3 no L2 promotion
    const uint8_t *g;
};
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

__global__ void __launch_bounds__(256, 1) stream(const __grid_constant__ CUtensorMap tm, P p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
    const int box_bytes = p.box_rows * 128 * p.kd;
    const int stage_bytes = box_bytes * p.boxes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + p.stages * stage_bytes);
    uint64_t *empty = full + p.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
        for (int s = 0; s < p.stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(p.mode == 5 ? 1 : p.nprod));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(p.csize));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (p.csize > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t rank = p.csize > 1 ? ctarank() : 0;
    const int cid = blockIdx.x / p.csize;
    const int row0 = (cid * p.box_rows * p.boxes) % (p.rows_total - p.box_rows * p.boxes);
    long long t0 = clock64();
    if (lane == 0 && warp >= 2 && warp < 2 + p.nprod) {
        const int w = warp - 2;
        int nb = 0;
        for (int b = w; b < p.boxes; b += p.nprod) ++nb;
        for (int it = 0; it < p.iters; ++it) {
            const int s = it % p.stages;
            if (p.mode == 5 && (it % p.nprod) != w) continue;     // producer w owns stages w, w + nprod, ...
            if (it >= p.stages) wait(&empty[s], ((it / p.stages) & 1) ^ 1);
            // every CTA's full barrier expects the whole stage (multicast boxes land from peers)
            asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                         "r"(p.mode == 5 ? p.boxes * box_bytes : (p.csize > 1 ? (w == 0 ? p.boxes * box_bytes : 0) : nb * box_bytes)) : "memory");
            const int kb = (it * p.kd) % p.kblocks;
            if (p.csize > 1) {
                for (int b = w; b < p.boxes; b += p.nprod) {
                    if (b % p.csize != (int)rank) continue;
                    uint8_t *dst = sm + s * stage_bytes + b * box_bytes;
                    const int r = row0 + b * p.box_rows;
                    const uint16_t mask = (uint16_t)((1u << p.csize) - 1);
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;"
                                 ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(r), "r"(kb), "h"(mask) : "memory");
                }
                continue;
            }
            for (int b = (p.mode == 5 ? 0 : w); b < p.boxes; b += (p.mode == 5 ? 1 : p.nprod)) {
                uint8_t *dst = sm + s * stage_bytes + b * box_bytes;
                const int r = row0 + b * p.box_rows;
                if (p.mode == 2) {
                    const uint8_t *src = p.g + ((size_t)r * 2048 + (size_t)kb * box_bytes) % ((size_t)p.rows_total * 2048 - box_bytes);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(su32(dst)), "l"((uint64_t)src), "r"(box_bytes), "r"(su32(&full[s])) : "memory");
                } else if (p.kd > 1)
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                                 ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(r), "r"(kb) : "memory");
                else
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                                 ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(r), "r"(kb) : "memory");
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int it = 0; it < p.iters; ++it) {
            const int s = it % p.stages;
            if (p.mode == 1) {
                asm volatile("{\n.reg .pred p;\nW1: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(su32(&full[s])), "r"((it / p.stages) & 1) : "memory");
            } else {
                wait(&full[s], (it / p.stages) & 1);
            }
            if (p.csize > 1) {
                for (int c = 0; c < p.csize; ++c) {     // release the stage in every CTA of the cluster
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(&empty[s])), "r"(c));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
                }
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
        }
        p.out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (p.csize > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
    const int rows = 32768, cols = 1024;          // 64 MB bf16
    void *buf;
    CK(cudaMalloc(&buf, (size_t)rows * cols * 2));
    CK(cudaMemset(buf, 1, (size_t)rows * cols * 2));
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    long long *out;
    CK(cudaMalloc(&out, 148 * 8));
    CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    CK(cudaMemset(out, 0, 148 * 8));
    printf("box_rows kd box_KB boxes stage_KB stages ring_KB nprod | B/clk/SM med (min)\n");
    struct C { int box_rows, kd, boxes, stages, nprod, csize = 1, mode = 0; };
    std::vector<C> cs = {
        {128, 1, 1, 12, 2, 1, 5}, {128, 1, 1, 12, 4, 1, 5}, {128, 1, 2, 6, 2, 1, 5}, {128, 1, 2, 6, 3, 1, 5},
        {128, 2, 2, 3, 3, 1, 5},
        {128, 1, 1, 12, 1, 1, 4}, {128, 1, 2, 6, 1, 1, 4}, {128, 2, 2, 3, 1, 1, 4}, {128, 2, 1, 6, 1, 1, 4},
        {128, 1, 1, 12, 1, 1, 0}, {128, 1, 1, 12, 1, 1, 1}, {128, 1, 1, 12, 1, 1, 2}, {128, 1, 1, 12, 1, 1, 3},
        {128, 1, 2, 6, 1, 1, 0}, {128, 1, 2, 6, 1, 1, 1}, {128, 1, 2, 6, 1, 1, 2}, {128, 1, 2, 6, 1, 1, 3},
        {128, 1, 4, 3, 1, 1, 2}, {128, 2, 2, 3, 1, 1, 3},
        {128, 1, 1, 12, 1}, {128, 1, 1, 6, 1}, {128, 1, 1, 3, 1}, {64, 1, 1, 12, 1},   // 16 / 8 KB stages
        {64, 1, 2, 6, 1}, {128, 1, 2, 3, 1},                                          // 16 / 32 KB, shallow
        {128, 2, 2, 3, 2, 2}, {128, 1, 4, 3, 2, 2}, {128, 1, 4, 3, 2, 4}, {128, 2, 4, 1, 2, 4},
        {128, 1, 2, 6, 2, 2}, {128, 2, 2, 2, 2, 2},
        {128, 1, 3, 4, 2}, {128, 3, 1, 4, 1},            // 48 KB stages
        {128, 3, 2, 2, 2}, {128, 1, 6, 2, 2},            // 96 KB stages
        {128, 2, 4, 1, 2},                               // one 128 KB stage (no pipelining)
        {128, 2, 3, 2, 2}, {128, 1, 5, 2, 2},            // 96 / 80 KB stages
        {128, 1, 2, 6, 1}, {128, 1, 2, 6, 2},            // 32 KB stages of two 16 KB boxes (kd = 1 GEMM)
        {128, 2, 1, 6, 1},                               // 32 KB stages, one 3-D box
        {128, 2, 2, 3, 1}, {128, 2, 2, 3, 2},            // 64 KB stages of two 32 KB boxes (kd = 2 GEMM)
        {128, 1, 4, 3, 2}, {128, 1, 4, 3, 4},            // 64 KB stages of four 16 KB boxes
        {128, 1, 2, 4, 2}, {128, 2, 2, 2, 2},            // smaller rings (128 KB)
        {128, 4, 1, 6, 1}, {128, 4, 2, 3, 2},            // 64 KB boxes
        {64, 2, 4, 3, 2}, {256, 1, 2, 3, 2},
    };
    for (auto c : cs) {
        CUtensorMap tm;
        cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
        cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
        if (c.mode == 4) {            // contiguous: row r of k-block kb at (kb * rows + r) * 128 B
            strides[0] = 128;
            strides[1] = (cuuint64_t)rows * 128;
        }
        cuuint32_t box[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.kd}, es[3] = {1, 1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, c.mode == 3 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            continue;
        }
        const int box_bytes = c.box_rows * 128 * c.kd, stage_bytes = box_bytes * c.boxes;
        const size_t smem = 1024 + (size_t)c.stages * stage_bytes + 256;
        if (smem > 232448) { printf("skip (smem)\n"); continue; }
        P p{c.stages, c.boxes, c.nprod, 1024, c.box_rows, c.kd, rows, cols / 64, out, c.csize, c.mode, (const uint8_t *)buf};
        const int grid = 148 / c.csize * c.csize;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 3; ++rep) CK(cudaLaunchKernelEx(&cfg, stream, tm, p));
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(grid);
        CK(cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost));
        std::sort(h.begin(), h.end());
        const double bytes = (double)p.iters * stage_bytes;
        printf("%8d %2d %6d %5d %8d %6d %7d %5d | %6.1f (%6.1f)\n", c.box_rows, c.kd, box_bytes / 1024, c.boxes,
               stage_bytes / 1024, c.stages, c.stages * stage_bytes / 1024, c.nprod, bytes / h[grid / 2], bytes / h[grid - 1]);
        printf("        mode %d\n", c.mode);
        if (c.csize > 1) printf("        (cluster %d, multicast: L2 reads per SM = %.1f B/clk)\n", c.csize, bytes / c.csize / h[grid / 2]);
    }
    return 0;
}
