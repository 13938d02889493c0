// Experiment: cost of issuing TMA loads from ONE thread, with no global stores in the issue
// loop (the earlier tma_ingest.cu stored a timestamp per stage, and the next stage's
// release-semantics expect_tx then waited for that store).  One CTA per SM; thread 0 arms one
// mbarrier with the total bytes, issues n boxes of {64 cols, rows} bf16 (128-B swizzle) back
// to back into distinct smem buffers, then waits.  Reports per CTA: clocks spent in the issue
// loop, clocks until completion, and bytes/clk.  Data: 256 MB buffer; "warm" = same 64 MB
// region read on the previous launch (L2-resident), "cold" = a fresh region each launch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_issue tma_issue.cu
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

struct P {
    int n, rows, row0, rows_total;
    long long *out;   // per CTA: [0] issue clk, [1] complete clk
};

__global__ void __launch_bounds__(128) issue(const __grid_constant__ CUtensorMap tm, P p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int box_bytes = p.rows * 128;
        const int r0 = (p.row0 + blockIdx.x * p.rows * 8) % p.rows_total;
        long long t0 = clock64();
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(p.n * box_bytes) : "memory");
        for (int i = 0; i < p.n; ++i) {
            const int c0 = (i % 16) * 64, c1 = (r0 + (i / 16) * p.rows) % p.rows_total;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su32(sm + i * box_bytes)), "l"((uint64_t)&tm), "r"(su32(&bar)), "r"(c0), "r"(c1) : "memory");
        }
        long long t1 = clock64();
        asm volatile("{\n.reg .pred q;\nW: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n@!q bra W;\n}" ::"r"(su32(&bar)) : "memory");
        long long t2 = clock64();
        p.out[2 * blockIdx.x] = t1 - t0;
        p.out[2 * blockIdx.x + 1] = t2 - t0;
    }
}

int main() {
    const int rows = 131072, cols = 1024;          // 256 MB bf16
    void *buf;
    CK(cudaMalloc(&buf, (size_t)rows * cols * 2));
    CK(cudaMemset(buf, 1, (size_t)rows * cols * 2));
    void *flush;
    CK(cudaMalloc(&flush, 512u << 20));
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    long long *out;
    CK(cudaMalloc(&out, 148 * 2 * 8));
    CK(cudaFuncSetAttribute(issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    printf("grid box_rows n KB | issue clk (med/max) | complete clk (med/max) | B/clk/SM med | mode\n");
    for (int cold = 0; cold < 2; ++cold)
        for (int box_rows : {64, 128, 256})
            for (int n : {1, 2, 4, 8, 12})
                for (int grid : {1, 148}) {
                    const int kb = n * box_rows * 128 / 1024;
                    if (kb > 192) continue;
                    CUtensorMap tm;
                    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
                    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
                    cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
                    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                        printf("encode failed\n");
                        continue;
                    }
                    std::vector<long long> h(2 * grid);
                    std::vector<long long> iss, cmp;
                    for (int rep = 0; rep < 6; ++rep) {
                        int row0 = cold ? (rep * 8192) % rows : 0;
                        if (cold) CK(cudaMemset(flush, rep, 512u << 20));
                        P p{n, box_rows, row0, rows, out};
                        issue<<<grid, 128, 1024 + n * box_rows * 128>>>(tm, p);
                        CK(cudaDeviceSynchronize());
                        CK(cudaMemcpy(h.data(), out, 16 * grid, cudaMemcpyDeviceToHost));
                        if (rep >= 2)
                            for (int b = 0; b < grid; ++b) { iss.push_back(h[2 * b]); cmp.push_back(h[2 * b + 1]); }
                    }
                    std::sort(iss.begin(), iss.end());
                    std::sort(cmp.begin(), cmp.end());
                    const double med = (double)cmp[cmp.size() / 2];
                    printf("%4d %4d %3d %4d | %6lld %6lld | %7lld %7lld | %6.1f | %s\n", grid, box_rows, n, kb, iss[iss.size() / 2],
                           iss.back(), cmp[cmp.size() / 2], cmp.back(), n * box_rows * 128 / med, cold ? "cold" : "warm");
                }
    return 0;
}
