// Weight-streaming tcgen05 dense for few (feature tile, token tile) units (DISPATCH.md
// family 4: bf16 dense_dyn with M <= 128, or M <= 1024 where the tiles leave most SMs idle;
// Nimble §3.5 residue dispatch PAPER.md:383-390).  With few tiles every weight byte feeds few
// tokens and one CTA per tile would use a handful of SMs, so the kernel splits K over S CTAs
// per tile and spreads the weight stream over most SMs.
//
// Grid = S x m_tiles x n_tiles CTAs; the S CTAs of a (feature tile, token tile) unit form one
// thread-block cluster along K (S <= 8, portable).  CTA (q, mt, nt) owns weight rows [128 mt, +128),
// tokens [128 nt, +128) and the k-blocks [q kb / S, (q+1) kb / S) (S depends on (N, K) and
// the token-tile count only, so a token's result is the same for M and for M padded to a
// multiple of 128: dynamic M == pad-then-slice, bit for bit).
//   warp 0 lane 0  TMA producer: the CTA's weight k-blocks are requested BEFORE the PDL
//                  grid-dependency wait (they overlap the previous kernel), the token
//                  k-blocks after it; rows >= M are zero-filled by TMA bounds.
//   warp 1         TMEM allocation; lane 0 issues tcgen05.mma (M = 128, N = 128, or on the
//                  last token tile the residue variant's width 16 ceil(r/16) / 128 for the
//                  fallback) into one fp32 accumulator.
//   all 8 warps    drain TMEM (warp w: lane quarter w % 4, token half w / 4) into this CTA's
//                  fp32 partial slab part[nt][mt][q][token][128] in L2 (128-B warp stores), one
//                  cluster barrier (release / acquire at cluster
//                  scope: ~0.1 us, where a global-memory flag barrier measured ~2 us on B200,
//                  scripts/exp/pdl_floor.cu), then CTA q reduces tokens j = q, q + S, ...: a
//                  thread takes (token, 4-feature) items, loads all S partials at once and sums
//                  them in split order 0..S-1 (deterministic), applies the epilogue (alpha |
//                  bias | bias+GELU | bias+residual) and stores bf16.
// The partial slab workspace is per stream; the next launch writes it only after its PDL
// grid-dependency wait, i.e. after this launch has completed.
#include "launch.h"
#include "ptx.cuh"

namespace nimble {

namespace {

constexpr int kWsThreads = 256;
constexpr int kWsWarps = kWsThreads / 32;
constexpr int kBK = 64;                       // one 128-B swizzle row of bf16
constexpr int kAB = 128 * kBK * 2;            // 16 KB weight k-block
constexpr int kWsMaxSplit = 16;               // cluster size limit (non-portable)

__device__ __forceinline__ float4 ldcg4(const float *p) { return __ldcg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void add4(float4 &a, const float4 &v) { a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w; }

template <int EPI>
__device__ __forceinline__ float epi1(float a, const WsParams &p, int f, int j) {
    if constexpr (EPI == 0) return a * p.alpha;
    a += __ldg(p.bias + f);
    if constexpr (EPI == 2) a = ptx::gelu_erf(a);
    if constexpr (EPI == 3) a += __bfloat162float(p.res[(size_t)j * p.ld_res + f]);
    return a;
}

__device__ __forceinline__ int S_of(const WsParams &p) { return p.S; }

template <int EPI>
__global__ void __launch_bounds__(kWsThreads, 2)    // two CTAs per SM: a PDL-overlapped neighbour fits
    ws_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const WsParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int b_bytes = p.n_box * 128;            // token k-block: n_box rows of 128 B
    const int stage_bytes = kAB + b_bytes;
    const int ring = (S_of(p) == 2 && p.stages * stage_bytes < p.n_box * 512) ? p.n_box * 512 : p.stages * stage_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + ring);   // after the ring (/ the S == 2 slab)
    uint64_t *empty = full + p.stages;
    uint64_t *tfull = empty + p.stages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    const int q = (int)blockIdx.x;                // rank in the K-split cluster
    const int mt = (int)blockIdx.y;               // 128-feature tile
    const int nt = (int)blockIdx.z;               // 128-token tile
    const int S = p.S;
    const int tok0 = nt * 128;
    int Mt = min(128, p.M - tok0);                // valid tokens of this token tile (device extent: below)
    uint32_t n_this = (nt == p.n_tiles - 1) ? (uint32_t)p.n_umma : 128u;   // residue width on the tail tile
    const int kb0 = (int)((int64_t)q * p.kb_total / S);
    const int kb1 = (int)((int64_t)(q + 1) * p.kb_total / S);
    const int nkb = kb1 - kb0;
    // debug timeline (kept in registers, written once at the end: no stores on the hot path)
    unsigned long long ts0 = 0, ts1 = 0, ts2 = 0, ts3 = 0, ts4 = 0, ts5 = 0;
    const bool tr = p.trace != nullptr;
    if (tr) ts0 = ptx::globaltimer();

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, 128);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();                                // the next kernel's prologue may start
    if (tr) ts1 = ptx::globaltimer();
    if (p.m_dev) {
        // device extent (one token tile): the residue dispatch of DISPATCH.md family 4 on the
        // device — every role but the producer (which waits in its own path) reads M here
        if (!(warp == 0 && lane == 0)) ptx::pdl_wait();   // (the producer waits in its own path)
        const int Md = warp == 0 && lane == 0 ? 0 : *p.m_dev;
        if (!(warp == 0 && lane == 0)) {
            if (Md < 1 || Md > p.M) __trap();          // outside [1, M_max]: caller bug, fail loudly
            const int r = Md % 128, k = Md / 128;
            const int cls = (r + 15) / 16, ncls = 9;
            const int cc = (p.var_c <= 0 || p.var_c >= ncls) ? ncls : p.var_c;
            const int variant = (cc == ncls || cls < cc - 1) ? cls : -1;
            Mt = Md;
            n_this = r ? (variant >= 0 ? 16u * (uint32_t)cls : 128u) : 128u;
            if (p.rec && threadIdx.x == 32 && blockIdx.x == 0 && blockIdx.y == 0) {
                nimble_dispatch d{};
                d.family = 4; d.tile_t = 128; d.granule = 16; d.n_classes = ncls; d.residue_class = cls;
                d.variant = variant; d.split_k = S; d.umma_m = 128; d.umma_n_full = 128;
                d.umma_n_tail = r ? (int32_t)n_this : 0; d.k = k; d.r = r;
                d.grid[0] = p.m_tiles; d.grid[1] = 1; d.grid[2] = S;
                d.cluster[0] = d.cluster[1] = d.cluster[2] = 1;
                *p.rec = d;
            }
        }
    }

    if (warp == 0 && lane == 0) {
        // ---- producer: weights first (static: before the grid-dependency wait), tokens after
        const int pre = nkb < p.stages ? nkb : p.stages;
        for (int i = 0; i < pre; ++i) {
            ptx::mbar_arrive_expect_tx_relaxed(&full[i], (uint32_t)stage_bytes);
            ptx::tma_load_3d(smem + i * stage_bytes, &tmA, &full[i], (kb0 + i) * kBK, mt * 128, 0);
        }
        ptx::pdl_wait();
        if (tr) ts2 = ptx::globaltimer();
        for (int i = 0; i < pre; ++i)
            ptx::tma_load_3d(smem + i * stage_bytes + kAB, &tmB, &full[i], (kb0 + i) * kBK, tok0, 0);
        for (int i = pre; i < nkb; ++i) {
            const int s = i % p.stages;
            ptx::mbar_wait(&empty[s], (uint32_t)(((i / p.stages) & 1) ^ 1));
            ptx::mbar_arrive_expect_tx_relaxed(&full[s], (uint32_t)stage_bytes);
            ptx::tma_load_3d(smem + s * stage_bytes, &tmA, &full[s], (kb0 + i) * kBK, mt * 128, 0);
            ptx::tma_load_3d(smem + s * stage_bytes + kAB, &tmB, &full[s], (kb0 + i) * kBK, tok0, 0);
        }
    } else if (warp == 1) {
        // ---- MMA issuer: the whole warp runs the loop converged, one elected lane issues (the
        // descriptors stay in uniform registers; a lane-0-only role wraps every tcgen05.mma in an
        // ELECT / R2UR.BROADCAST loop, umma_gemm.cu)
        const uint32_t idesc = ptx::idesc_bf16(128u, n_this, 0u);
        for (int i = 0; i < nkb; ++i) {
            const int s = i % p.stages;
            ptx::mbar_wait(&full[s], (uint32_t)((i / p.stages) & 1));
            ptx::tc_fence_after();
            const uint32_t sa = ptx::smem_u32(smem + s * stage_bytes);
            const uint64_t adesc = ptx::smem_desc_sw128(sa, 0, 1024);
            const uint64_t bdesc = ptx::smem_desc_sw128(sa + kAB, 0, 1024);
            if (ptx::elect_one()) {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                    ptx::umma_bf16(tmem_base, adesc + (uint64_t)((kk * 32) >> 4), bdesc + (uint64_t)((kk * 32) >> 4),
                                   idesc, (i > 0 || kk > 0) ? 1u : 0u);
                ptx::umma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::umma_commit(tfull);
        __syncwarp();
    }
    __syncwarp();
    if (p.m_dev) Mt = *p.m_dev;                        // every thread has passed the dependency wait

    // ---- drain the accumulator into this CTA's partial slab: TMEM lane = feature, so a warp's
    // store of one token covers 32 consecutive features (128 B).  (Transposing through shared
    // memory for 16-B stores measured slower: scripts/gpu_probe6.sh, NIMBLE_WS_FLAGS history.)
    const size_t slab = (size_t)p.n_box * 128;                  // floats per (tile, split) slab
    float *part_tile = p.part + ((size_t)nt * p.m_tiles + mt) * S * slab;
    {
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        if (tr) ts3 = ptx::globaltimer();
        const int quarter = (int)(warp & 3), half = (int)(warp >> 2);
        const int f = quarter * 32 + (int)lane;
        float *mine = part_tile + (size_t)q * slab;
        float *sp = reinterpret_cast<float *>(smem);  // S == 2: the slab stays in shared memory (ring is free)
        for (int c0 = half * 16; c0 < Mt; c0 += 32) {
            float v[16];
            ptx::tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
            if (S == 2) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < Mt) sp[(c0 + j) * 128 + f] = v[j];
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < Mt) __stcg(mine + (size_t)(c0 + j) * 128 + f, v[j]);
            }
        }
        ptx::tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {                                   // TMEM free for a co-resident next kernel
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 128);
    }
    if (tr) ts4 = ptx::globaltimer();
    ptx::cluster_arrive();                             // release: the slab is written
    ptx::cluster_wait();                               // acquire: every split's slab is visible
    if (tr) ts5 = ptx::globaltimer();

    // ---- reduction over the S splits of this tile (fixed order 0..S-1) + epilogue.  CTA q owns
    // tokens q, q + S, ...; its threads take (token, 4-feature quad) items and issue every
    // split's load of an item before summing (one L2 round trip per item).
    const int n_tok = Mt > q ? (Mt - q + S - 1) / S : 0;
    const int items = n_tok * 32;
    for (int it = (int)threadIdx.x; it < items; it += kWsThreads) {
        const int jl = q + S * (it >> 5), l = it & 31;
        const float *src = part_tile + (size_t)jl * 128 + 4 * l;
        const int j = tok0 + jl;                          // output row
        float4 a;
        if (S == 2) {
            // the two slabs live in the two CTAs' shared memory: own + the peer's over DSMEM,
            // summed in split order (part 0 + part 1) as the L2 path does
            const uint32_t la = ptx::smem_u32(smem) + (uint32_t)((jl * 128 + 4 * l) * 4);
            const float4 own = *reinterpret_cast<const float4 *>(smem + (size_t)(jl * 128 + 4 * l) * 4);
            const float4 peer = ld_dsmem4(ptx::map_shared_rank(la, (uint32_t)(q ^ 1)));
            a = q == 0 ? own : peer;
            add4(a, q == 0 ? peer : own);
        } else {
            float4 v[kWsMaxSplit];
#pragma unroll
            for (int u = 0; u < kWsMaxSplit; ++u)
                v[u] = u < S ? ldcg4(src + (size_t)u * slab) : make_float4(0.f, 0.f, 0.f, 0.f);
            a = v[0];
#pragma unroll
            for (int u = 1; u < kWsMaxSplit; ++u)
                if (u < S) add4(a, v[u]);
        }
        const int f = mt * 128 + 4 * l;
        if (f >= p.N) continue;
        __nv_bfloat16 *dst = p.out + (size_t)j * p.ld_out + f;
        if (f + 4 <= p.N) {
            const float y0 = epi1<EPI>(a.x, p, f, j), y1 = epi1<EPI>(a.y, p, f + 1, j);
            const float y2 = epi1<EPI>(a.z, p, f + 2, j), y3 = epi1<EPI>(a.w, p, f + 3, j);
            __nv_bfloat162 o0 = __floats2bfloat162_rn(y0, y1), o1 = __floats2bfloat162_rn(y2, y3);
            uint2 o;
            o.x = *reinterpret_cast<uint32_t *>(&o0);
            o.y = *reinterpret_cast<uint32_t *>(&o1);
            *reinterpret_cast<uint2 *>(dst) = o;
        } else {                                        // ragged feature tail (N % 4 != 0)
            const float av[4] = {a.x, a.y, a.z, a.w};
            for (int e = 0; e < 4 && f + e < p.N; ++e) dst[e] = __float2bfloat16_rn(epi1<EPI>(av[e], p, f + e, j));
        }
    }
    if (S == 2) {                                      // the peer may still read this CTA's slab
        ptx::cluster_arrive();
        ptx::cluster_wait();
    }
    if (tr && threadIdx.x == 0) {
        unsigned long long *t = p.trace + (((size_t)nt * p.m_tiles + mt) * S + q) * 8;
        t[0] = ts0; t[1] = ts1; t[2] = ts2; t[3] = ts3; t[4] = ts4; t[5] = ts5; t[6] = ptx::globaltimer();
    }
}

template <int EPI>
cudaError_t launch_ws_t(const WsLaunch &L) {
    auto fn = ws_gemm_kernel<EPI>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)L.p.S, (unsigned)L.p.m_tiles, (unsigned)L.p.n_tiles);
    cfg.blockDim = dim3(kWsThreads, 1, 1);
    cfg.dynamicSmemBytes = L.smem_bytes;
    cfg.stream = L.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)L.p.S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.numAttrs = 1;
    if (pdl_enabled()) {
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
    cfg.attrs = at;
    return cudaLaunchKernelEx(&cfg, fn, L.tmA, L.tmB, L.p);
}

}  // namespace

size_t ws_smem_bytes(int n_box, int stages, int S) {
    // S == 2: the ring doubles as the fp32 [tokens][128] partial slab exchanged over DSMEM
    size_t ring = (size_t)stages * (kAB + (size_t)n_box * 128);
    if (S == 2 && ring < (size_t)n_box * 512) ring = (size_t)n_box * 512;
    return 1024 /* alignment slack */ + ring + 256 /* barriers, TMEM slot */;
}

// Can a cluster of S CTAs of this size be scheduled at all on this device (under MPS / green
// contexts an SM partition may be smaller than a cluster)?
bool ws_cluster_fits(int S, size_t smem_bytes) {
    auto fn = ws_gemm_kernel<1>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)S, 1, 1);
    cfg.blockDim = dim3(kWsThreads, 1, 1);
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = (unsigned)S;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return n >= 1;
}

cudaError_t launch_ws_gemm(const WsLaunch &L) {
    switch (L.epi) {
        case 0: return launch_ws_t<0>(L);
        case 1: return launch_ws_t<1>(L);
        case 2: return launch_ws_t<2>(L);
        default: return launch_ws_t<3>(L);
    }
}

}  // namespace nimble
