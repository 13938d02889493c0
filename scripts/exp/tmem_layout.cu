// Experiment: the register <-> TMEM mapping of tcgen05.ld.16x256b (one warp, lanes 0-31,
// columns 0-15 filled with value = 1000 * lane + column by 32x32b stores).
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t *out) {
    __shared__ uint32_t slot;
    const int lane = threadIdx.x;
    if (threadIdx.x < 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = 1000u * lane + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(base), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(base));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
    uint32_t s[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7]) : "r"(base + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[128 + lane * 8 + i] = s[i];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}
int main() {
    uint32_t *d, h[384];
    cudaMalloc(&d, sizeof(h));
    k<<<1, 32>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %d\n16x256b.x1 @lane0 (value = 1000*lane + col):\n", (int)e);
    for (int t = 0; t < 32; ++t) printf("t%02d: %5u %5u %5u %5u\n", t, h[t * 4], h[t * 4 + 1], h[t * 4 + 2], h[t * 4 + 3]);
    printf("16x256b.x2 @lane16:\n");
    for (int t = 0; t < 8; ++t) {
        printf("t%02d:", t);
        for (int i = 0; i < 8; ++i) printf(" %5u", h[128 + t * 8 + i]);
        printf("\n");
    }
}
