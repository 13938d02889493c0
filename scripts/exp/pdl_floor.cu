// Experiment: the per-launch floor of a dependent kernel chain on B200 (CUDA graph of 20
// launches, with / without programmatic dependent launch).  Each kernel reads one value the
// previous one wrote and writes one value (a true dependency), so the chain is serial.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_floor pdl_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

template <int MODE>
__global__ void chain(float *buf, int i, unsigned *bar, int G) {
    // MODE 0: read prev, write next.  MODE 1: + grid barrier (atomic + spin) before the write.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float v = 0.f;
    if (threadIdx.x == 0) v = __ldcg(buf + (i & 1));
    if (MODE == 1) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned g0;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(bar + 1) : "memory");
            unsigned t = atomicAdd(bar, 1u);
            if (t == (unsigned)G - 1) {
                *(volatile unsigned *)bar = 0u;
                __threadfence();
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
            } else {
                while (true) {
                    unsigned g;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
                    if (g != g0) break;
                }
            }
        }
        __syncthreads();
    }
    if (MODE == 2 || MODE == 3) {
        // relaxed polling, one acquire fence after; release atomic arrive.  MODE 3: groups of
        // 16 consecutive CTAs (per-tile barrier), each group its own (count, gen) pair.
        const int grp = MODE == 3 ? blockIdx.x / 16 : 0;
        const int gsz = MODE == 3 ? min(16, G - grp * 16) : G;
        unsigned *c = bar + 2 + 2 * grp;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned g0;
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(c + 1) : "memory");
            unsigned t;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(c) : "memory");
            if (t == (unsigned)gsz - 1) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(c) : "memory");
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c + 1) : "memory");
            } else {
                while (true) {
                    unsigned g;
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(c + 1) : "memory");
                    if (g != g0) break;
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    if (MODE == 4) {            // cluster barrier (the launch sets a cluster of 8)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) buf[(i + 1) & 1] = v + 1.f;
}

template <int MODE>
float run(int grid, int block, bool pdl, float *buf, unsigned *bar) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 20; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (pdl) {
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        if (MODE == 4) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = 8; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1;
            ++na;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        CK(cudaLaunchKernelEx(&cfg, chain<MODE>, buf, i, bar, grid));
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, s));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, s);
        CK(cudaGraphLaunch(ge, s));
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best * 1e3f / 20.f;
}

int main() {
    float *buf;
    unsigned *bar;
    CK(cudaMalloc(&buf, 8));
    CK(cudaMalloc(&bar, 4096));
    CK(cudaMemset(buf, 0, 8));
    CK(cudaMemset(bar, 0, 4096));
    printf("per-launch us (graph of 20 dependent launches)\n");
    for (int grid : {8, 24, 128, 144})
        for (int pdl = 0; pdl < 2; ++pdl) {
            printf("grid %3d pdl %d : plain %.2f  | +grid barrier %.2f | relaxed poll %.2f | groups of 16 %.2f | cluster-8 barrier %.2f\n",
                   grid, pdl, run<0>(grid, 256, pdl, buf, bar), run<1>(grid, 256, pdl, buf, bar),
                   run<2>(grid, 256, pdl, buf, bar), run<3>(grid, 256, pdl, buf, bar),
                   grid % 8 == 0 ? run<4>(grid, 256, pdl, buf, bar) : -1.f);
        }
    return 0;
}
