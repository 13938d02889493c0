// Hand-written inline-PTX wrappers for sm_100a: mbarrier, TMA (cp.async.bulk.tensor),
// tcgen05 (alloc / mma / commit / ld / fences), cluster / DSMEM.
// Written from the PTX ISA semantics; no CUTLASS/CuTe code is used.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace nimble {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }

// ----------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// relaxed form for producers that publish nothing but the TMA bytes themselves (tracked by
// complete_tx): a release arrive would first wait for the thread's earlier global stores.
__device__ __forceinline__ void mbar_arrive_expect_tx_relaxed(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a protocol bug becomes a trap (launch error) instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins == (1u << 26)) __trap();
    }
}

// ----------------------------------------------------------------- TMA
// TMA tile prefetch into L2 (no smem destination, no barrier): warms the box for a later load.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *m, int32_t c0, int32_t c1, int32_t c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 3-D tiled bulk tensor load global -> shared, completion on an mbarrier (complete_tx)
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// ----------------------------------------------------------------- tcgen05
// TMEM allocation: ncols power of two >= 32; the address lands in smem.
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// One lane of a converged warp (elect.sync): the MMA issuer runs its loop with the whole warp
// converged so the descriptors stay warp-uniform (uniform registers, no per-MMA R2UR loop).
__device__ __forceinline__ bool elect_one() {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok));
    return ok != 0;
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate), one CTA.
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on an mbarrier once every prior tcgen05 async op of this thread completes.
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 bits, 16 consecutive columns: thread t of the warp gets lane (base+t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Split form: several loads in flight, then one wait.  tmem_wait16 names the registers as
// in/out operands of the wait, so no use of them can be scheduled above it.
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"):
//   [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1 (sm_100),
//   [49,52) base offset 0, bit 52 LBO mode 0, [61,64) layout: 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// Instruction descriptor, kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// A K-major (bit 15 = 0), B major bit 16, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ __forceinline__ uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ----------------------------------------------------------------- cluster / DSMEM
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_shared_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ float ld_shared_cluster_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

// ----------------------------------------------------------------- math
// GELU(z) = z/2 (1 + erf(z / sqrt 2)).
// erf_as26: Abramowitz & Stegun 7.1.26 (max abs error 1.5e-7): one exp2 + one rcp (2 MUFU).
// erf_as28: Abramowitz & Stegun 7.1.28, erf(x) = 1 - (1 + a1 x + ... + a6 x^6)^-16 (max abs
//           error 2.6e-7 in exact arithmetic, ~2e-6 in fp32): one rcp + FMAs (1 MUFU op).
// Both are far below the bf16 output rounding (2^-9 relative) of the fused epilogue.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float erf_as26(float x) {
    const float ax = fabsf(x);
    const float t = rcp_approx(fmaf(0.3275911f, ax, 1.0f));
    float poly = fmaf(1.061405429f, t, -1.453152027f);
    poly = fmaf(poly, t, 1.421413741f);
    poly = fmaf(poly, t, -0.284496736f);
    poly = fmaf(poly, t, 0.254829592f);
    poly *= t;
    const float e = exp2f(-ax * ax * 1.4426950408889634f);
    return copysignf(fmaf(-poly, e, 1.0f), x);
}
__device__ __forceinline__ float erf_as28(float x) {
    const float ax = fminf(fabsf(x), 8.0f);
    float p = fmaf(4.30638e-5f, ax, 2.765672e-4f);
    p = fmaf(p, ax, 1.520143e-4f);
    p = fmaf(p, ax, 9.2705272e-3f);
    p = fmaf(p, ax, 4.22820123e-2f);
    p = fmaf(p, ax, 7.05230784e-2f);
    p = fmaf(p, ax, 1.0f);
    float r = rcp_approx(p);
    r *= r; r *= r; r *= r; r *= r;                  // p^-16
    return copysignf(1.0f - r, x);
}
#ifdef NIMBLE_ERF_AS26
__device__ __forceinline__ float erf_as(float x) { return erf_as26(x); }
#else
__device__ __forceinline__ float erf_as(float x) { return erf_as28(x); }
#endif
#ifdef NIMBLE_GELU_ERFF
__device__ __forceinline__ float gelu_erf(float z) { return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f)); }
#elif defined(NIMBLE_GELU_UNFOLDED)
__device__ __forceinline__ float gelu_erf(float z) { return 0.5f * z * (1.0f + erf_as(z * 0.70710678118654752f)); }
#else
// GELU(z) = z Phi(z), Phi(z) = (1 + erf(z / sqrt2)) / 2, with erf from A&S 7.1.28 (the same
// approximation as erf_as28, |error| <= 5e-7 on GELU) re-associated for the epilogue's issue
// budget (14 instructions, two MUFU; the epilogue of the GELU GEMM is issue-bound):
//   * 1/sqrt2 is folded into the coefficients (b_i = a_i 2^(-i/2)),
//   * the 1/2 of Phi is folded in too: scaling p by 2^(1/16) gives h = p^-16 = (1 - erf) / 2,
//   * Phi = 1 - h (z >= 0) or h (z < 0), so z Phi = max(z, 0) - |z h| with no select,
//   * p^-16 = rcp(p)^16 (rcp.approx relative error ~2^-23, x16 -> ~2e-6 relative on h; the
//     former ex2(-16 lg2 p) form, NIMBLE_GELU_LG2EX2, costs two MUFU per value).
__device__ __forceinline__ float gelu_erf(float z) {
    const float q = fabsf(z);
    float p = fmaf(5.621299664e-06f, q, 5.105520901e-05f);
    p = fmaf(p, q, 3.968613701e-05f);
    p = fmaf(p, q, 3.422739239e-03f);
    p = fmaf(p, q, 2.207699846e-02f);
    p = fmaf(p, q, 5.207516304e-02f);
    p = fmaf(p, q, 1.044273782e+00f);
#ifndef NIMBLE_GELU_LG2EX2
    float h = rcp_approx(p);                         // p^-16 = rcp(p)^16: one MUFU + four squarings
    h *= h; h *= h; h *= h; h *= h;                  // 2^-1 (1 + sum a_i x^i)^-16
#else
    float h;                                         // p^-16 = 2^(-16 log2 p): 3 instructions, 2 MUFU
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(h) : "f"(p));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(h) : "f"(-16.0f * h));
#endif
    return fmaxf(z, 0.0f) - fabsf(z * h);
}
#endif
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2) and the 3-input max (FMNMX3).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// gelu_erf on two values at once: the same arithmetic as gelu_erf (same constants, same
// order per element), with the polynomial and products in FFMA2 / FMUL2.
__device__ __forceinline__ float2 gelu_erf2(float2 z) {
    const float2 q = make_float2(fabsf(z.x), fabsf(z.y));
    float2 p = ffma2(f2(5.621299664e-06f), q, f2(5.105520901e-05f));
    p = ffma2(p, q, f2(3.968613701e-05f));
    p = ffma2(p, q, f2(3.422739239e-03f));
    p = ffma2(p, q, f2(2.207699846e-02f));
    p = ffma2(p, q, f2(5.207516304e-02f));
    p = ffma2(p, q, f2(1.044273782e+00f));
    float2 h;
#if defined(NIMBLE_GELU_NR)                          // experiment: measured 4 % slower (FMA issue)
    // 1/p without MUFU: magic-constant estimate (|rel err| < 0.125 for p >= 1) + 3 Newton steps
    // (rel err ~ 3e-8) on the FMA pipes, then p^-16 by squaring
    h = make_float2(__int_as_float(0x7EF311C3 - __float_as_int(p.x)), __int_as_float(0x7EF311C3 - __float_as_int(p.y)));
#pragma unroll
    for (int it = 0; it < 3; ++it) {
        const float2 e = ffma2(make_float2(-p.x, -p.y), h, f2(1.0f));
        h = ffma2(h, e, h);
    }
    h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h);
#elif defined(NIMBLE_GELU_RCP2)
    // one MUFU per TWO values: r = 1 / (p.x p.y), 1/p.x = r p.y, 1/p.y = r p.x (two more roundings:
    // ~2^-22 relative on 1/p, x16 -> ~4e-6 on h; GELU(-1) is 2.5e-4 from a bf16 midpoint)
    {
        const float r = rcp_approx(p.x * p.y);
        h = fmul2(f2(r), make_float2(p.y, p.x));
    }
    h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h);
#elif !defined(NIMBLE_GELU_LG2EX2)
    // one MUFU per value and p^-16 by squaring: half the MUFU traffic of lg2 + ex2, which the
    // GELU GEMM's main loop felt (stage interval 1278 -> 1149 clk, FFN1 at M = 17448
    // 123.5 -> 120.6 us, scripts/trace_stages.py); rcp.approx's 2^-23 error x16 stays < 4e-6
    h = make_float2(rcp_approx(p.x), rcp_approx(p.y));
    h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h); h = fmul2(h, h);
#else
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(h.x) : "f"(p.x));
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(h.y) : "f"(p.y));
    h = fmul2(h, f2(-16.0f));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(h.x) : "f"(h.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(h.y) : "f"(h.y));
#endif
    const float2 w = fmul2(z, h);
    return make_float2(fmaxf(z.x, 0.0f) - fabsf(w.x), fmaxf(z.y, 0.0f) - fabsf(w.y));
}
__device__ __forceinline__ float sigmoidf_(float z) { return 1.0f / (1.0f + expf(-z)); }

}  // namespace ptx
}  // namespace nimble

namespace nimble {
namespace ptx {
// ----------------------------------------------------------------- PDL (programmatic dependent launch)
// wait: block until the preceding grid in the stream has completed and its memory is visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// trigger: allow the next grid in the stream to be scheduled (its prologue overlaps our tail).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ----------------------------------------------------------------- TMA store (smem -> global, bulk group)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, const void *src, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *m, const void *src, int32_t c0, int32_t c1,
                                             int32_t c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
// ---- on-device tensor-map patching (sm_90a / sm_100a "modifiable TMA"): a 128-B map copied
// into shared memory gets one global_dim replaced, is written back to a global slot with a
// release fence to the tensormap proxy (warp-wide .sync.aligned), and a consumer acquires it.
template <int DIM>
__device__ __forceinline__ void tmap_replace_dim_smem(void *smem_map, uint32_t extent) {
    asm volatile("tensormap.replace.tile.global_dim.shared::cta.b1024.b32 [%0], %1, %2;" ::"r"(smem_u32(smem_map)),
                 "n"(DIM), "r"(extent)
                 : "memory");
}
__device__ __forceinline__ void tmap_cp_fence_release(void *gmem_map, const void *smem_map) {
    asm volatile(
        "tensormap.cp_fenceproxy.global.shared::cta.tensormap::generic.release.gpu.sync.aligned [%0], [%1], 128;" ::"l"(
            reinterpret_cast<uint64_t>(gmem_map)),
        "r"(smem_u32(smem_map))
        : "memory");
}
__device__ __forceinline__ void tmap_fence_acquire(const void *gmem_map) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(gmem_map))
                 : "memory");
}
// Copy a tensor map (param space) into smem, patch one extent, publish it to `slot` (global),
// acquire it.  Called by one full warp; returns the map to use for TMA.
template <int DIM>
__device__ __forceinline__ const CUtensorMap *tmap_patch_extent(const CUtensorMap *tmpl, void *smem_map,
                                                               CUtensorMap *slot, uint32_t extent, uint32_t lane) {
    if (lane < 8) reinterpret_cast<uint4 *>(smem_map)[lane] = reinterpret_cast<const uint4 *>(tmpl)[lane];
    __syncwarp();
    if (lane == 0) tmap_replace_dim_smem<DIM>(smem_map, extent);
    __syncwarp();
    tmap_cp_fence_release(slot, smem_map);
    tmap_fence_acquire(slot);
    return slot;
}

__device__ __forceinline__ void tma_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// DSMEM load without a compiler memory clobber so independent loads can be in flight together
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
}  // namespace ptx
}  // namespace nimble

namespace nimble {
namespace ptx {
// mbarrier arrive (count 1), local CTA
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// expect_tx without arriving (the arrive comes from someone else / later)
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// Bulk DSMEM copy: own smem -> a peer CTA's smem, completion (complete_tx) on the PEER's mbarrier.
// dst and bar are shared::cluster addresses (mapa).
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, const void *src, uint32_t bytes,
                                                  uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst_cluster),
        "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
        : "memory");
}
// 3-D TMA load with an mbarrier (same as tma_load_3d, named for the residual tile)
__device__ __forceinline__ void tma_load_3d_nb(void *dst, const CUtensorMap *m, uint64_t *bar, int32_t c0, int32_t c1,
                                               int32_t c2) {
    tma_load_3d(dst, m, bar, c0, c1, c2);
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
}  // namespace ptx
}  // namespace nimble

namespace nimble {
namespace ptx {
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
}  // namespace ptx
}  // namespace nimble

namespace nimble {
namespace ptx {
// ----------------------------------------------------------------- CTA pair (cta_group::2)
__device__ __forceinline__ void tmem_alloc_pair(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem of both CTAs] (+)= A[smem of both CTAs] * B[smem halves of both CTAs]^T, M = 256.
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the mbarrier at the same smem offset in every CTA of `mask` once prior MMAs finish.
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// TMA load whose completion bytes land on the EVEN CTA's barrier of the pair (peer bit cleared).
__device__ __forceinline__ void tma_load_3d_pair(void *dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                                 int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// Remote arrive on a barrier of another CTA in the cluster (address from mapa).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
}  // namespace ptx
}  // namespace nimble

namespace nimble {
namespace ptx {
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
}  // namespace ptx
}  // namespace nimble
