// sm_100a gather / scatter kernels of the Tokencake offload/upload hot path, and the synthetic-content fill kernel.
//
// Data movement only — no tensor cores (no contraction anywhere on this path).  One warp copies one
// (block, layer, K|V) chunk of C contiguous bytes with 16-byte vector loads/stores, U loads in flight per lane before
// the matching stores (Little's law against HBM / host-link latency).  Each CTA owns a contiguous range of chunks,
// stages that range's descriptors in shared memory once (one host-link round trip when the descriptors sit in mapped
// pinned memory), and the warp that copies chunk 0 of a block performs the fused block-table epilogue
// (P:649 location flag / remap).
#include "kernels.cuh"

namespace tc {
namespace {

constexpr int kUnroll = 8;

__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream(int4 *p, const int4 &v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// Copy nv int4 vectors; the warp's 32 lanes cover 512 contiguous bytes per step.
__device__ __forceinline__ void warp_copy(int4 *__restrict__ dst, const int4 *__restrict__ src, int64_t nv, int lane) {
    int64_t v = lane;
    for (; v + 32 * (kUnroll - 1) < nv; v += 32 * kUnroll) {
        int4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) r[u] = ld_stream(src + v + 32 * u);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) st_stream(dst + v + 32 * u, r[u]);
    }
    for (; v < nv; v += 32) st_stream(dst + v, ld_stream(src + v));
}

// Device-side launch timing (tc_timing): earliest CTA start / latest CTA end on the %globaltimer clock (ns), so a
// kernel's duration excludes host launch latency.  g.ts = {start, end}, pre-set to {UINT64_MAX, 0}; null = off.
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ts_begin(const XferGeom &g) {
    if (g.ts) atomicMin(g.ts, now_ns());
}
__device__ __forceinline__ void ts_end(const XferGeom &g) {
    if (g.ts) atomicMax(g.ts + 1, now_ns());
}

template <bool kGather>
__device__ __forceinline__ void xfer_body(const XferDesc *__restrict__ desc, int64_t n, const XferGeom &g,
                                          char *__restrict__ kv, int32_t *__restrict__ table, int64_t chunks_per_cta,
                                          XferDesc *sdesc) {
    const int64_t M = n * g.two_l;
    const int64_t j0 = (int64_t)blockIdx.x * chunks_per_cta;
    if (j0 >= M) return;
    if (threadIdx.x == 0) ts_begin(g);
    const int64_t j1 = min(M, j0 + chunks_per_cta);
    const int64_t i0 = j0 / g.two_l;
    const int nb = (int)((j1 - 1) / g.two_l - i0 + 1);
    {
        const int4 *s = reinterpret_cast<const int4 *>(desc + i0);
        int4 *d = reinterpret_cast<int4 *>(sdesc);
        for (int k = threadIdx.x; k < nb; k += blockDim.x) d[k] = s[k];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int64_t nv = g.chunk >> 4;
    for (int64_t j = j0 + warp; j < j1; j += nwarps) {
        const int64_t i = j / g.two_l;
        const int64_t lk = j - i * g.two_l;
        const XferDesc d = sdesc[i - i0];
        char *pool_chunk = kv + (lk * g.n_pool + d.blk) * g.chunk;
        char *ext_chunk = reinterpret_cast<char *>(d.ext) + lk * g.chunk;
        if (kGather)
            warp_copy(reinterpret_cast<int4 *>(ext_chunk), reinterpret_cast<const int4 *>(pool_chunk), nv, lane);
        else
            warp_copy(reinterpret_cast<int4 *>(pool_chunk), reinterpret_cast<const int4 *>(ext_chunk), nv, lane);
        if (lk == 0 && lane == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
    }
    if (g.ts) {
        __syncthreads();
        if (threadIdx.x == 0) ts_end(g);
    }
}

template <bool kGather>
__global__ void __launch_bounds__(256) k_xfer(const XferDesc *__restrict__ desc, int64_t n, XferGeom g,
                                              char *__restrict__ kv, int32_t *__restrict__ table,
                                              int64_t chunks_per_cta) {
    extern __shared__ XferDesc sdesc[];
    xfer_body<kGather>(desc, n, g, kv, table, chunks_per_cta, sdesc);
}

template <bool kGather>
__global__ void __launch_bounds__(256) k_xfer_inl(const __grid_constant__ InlineDescs descs, int32_t n, XferGeom g,
                                                  char *__restrict__ kv, int32_t *__restrict__ table,
                                                  int64_t chunks_per_cta) {
    __shared__ XferDesc sdesc[kMaxInlineDesc + 2];
    xfer_body<kGather>(descs.d, n, g, kv, table, chunks_per_cta, sdesc);
}

// ------------------------------------------------------------------------------------------------ TMA bulk variant
// One elected thread per CTA streams its chunk range through an NS-stage shared-memory ring with the TMA bulk-copy
// engine: cp.async.bulk global->shared (mbarrier complete_tx), then cp.async.bulk shared->global (bulk_group).
// Whole pieces of up to `piece` bytes move as single bulk transactions, to or from mapped host memory or HBM.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, const void *src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int kStages = 8;

template <bool kGather>
__global__ void __launch_bounds__(32) k_xfer_bulk(const XferDesc *__restrict__ desc, int64_t n, XferGeom g,
                                                  char *__restrict__ kv, int32_t *__restrict__ table,
                                                  int64_t chunks_per_cta, int32_t piece) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;                                                   // kStages x piece
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * piece);  // kStages mbarriers
    XferDesc *sdesc = reinterpret_cast<XferDesc *>(bars + kStages);
    const int64_t M = n * g.two_l;
    const int64_t j0 = (int64_t)blockIdx.x * chunks_per_cta;
    if (j0 >= M) return;
    const int64_t j1 = min(M, j0 + chunks_per_cta);
    const int64_t i0 = j0 / g.two_l;
    const int nb = (int)((j1 - 1) / g.two_l - i0 + 1);
    {
        const int4 *s = reinterpret_cast<const int4 *>(desc + i0);
        int4 *d = reinterpret_cast<int4 *>(sdesc);
        for (int k = threadIdx.x; k < nb; k += blockDim.x) d[k] = s[k];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    ts_begin(g);
    const int32_t ppc = (int32_t)((g.chunk + piece - 1) / piece);   // pieces per chunk
    const int64_t K = (j1 - j0) * ppc;
    auto locate = [&](int64_t k, char *&src, char *&dst, uint32_t &bytes) {
        const int64_t j = j0 + k / ppc;
        const int64_t off = (int64_t)(k % ppc) * piece;
        const int64_t i = j / g.two_l;
        const int64_t lk = j - i * g.two_l;
        const XferDesc d = sdesc[i - i0];
        char *pool_chunk = kv + (lk * g.n_pool + d.blk) * g.chunk + off;
        char *ext_chunk = reinterpret_cast<char *>(d.ext) + lk * g.chunk + off;
        bytes = (uint32_t)min((int64_t)piece, g.chunk - off);
        src = kGather ? pool_chunk : ext_chunk;
        dst = kGather ? ext_chunk : pool_chunk;
        if (lk == 0 && off == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
    };
    auto issue_load = [&](int64_t k) {
        char *src, *dst;
        uint32_t bytes;
        locate(k, src, dst, bytes);
        const int s = (int)(k % kStages);
        mbar_expect_tx(&bars[s], bytes);
        bulk_load(ring + (size_t)s * piece, src, bytes, &bars[s]);
    };
    for (int64_t k = 0; k < K && k < kStages; ++k) issue_load(k);
    for (int64_t k = 0; k < K; ++k) {
        const int s = (int)(k % kStages);
        mbar_wait(&bars[s], (uint32_t)((k / kStages) & 1));
        char *src, *dst;
        uint32_t bytes;
        const int64_t j = j0 + k / ppc;
        const int64_t off = (int64_t)(k % ppc) * piece;
        const int64_t i = j / g.two_l;
        const int64_t lk = j - i * g.two_l;
        const XferDesc d = sdesc[i - i0];
        dst = kGather ? reinterpret_cast<char *>(d.ext) + lk * g.chunk + off : kv + (lk * g.n_pool + d.blk) * g.chunk + off;
        bytes = (uint32_t)min((int64_t)piece, g.chunk - off);
        (void)src;
        bulk_store(dst, ring + (size_t)s * piece, bytes);
        bulk_commit();
        if (k >= 1 && k - 1 + kStages < K) {   // refill the previous stage once its store has read smem
            bulk_wait_read<1>();
            issue_load(k - 1 + kStages);
        }
    }
    bulk_wait_all();
    ts_end(g);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// One CTA per (layer*2+kv, block) chunk (grid-stride); words inside a chunk in [T][Hl][wpr] order.
__global__ void k_fill(uint64_t *__restrict__ kv, int64_t n_chunks, int64_t n_pool, int32_t T, int32_t H,
                       int32_t Hl, int32_t rank, int32_t wpr, uint64_t seedk) {
    const int32_t cw = T * Hl * wpr;  // words per chunk
    for (int64_t q = blockIdx.x; q < n_chunks; q += gridDim.x) {
        const uint64_t base = (uint64_t)q * (uint64_t)T;   // ((lk*N + b) * T) in the unsharded index
        uint64_t *dst = kv + q * (int64_t)cw;
        for (int32_t w = threadIdx.x; w < cw; w += blockDim.x) {
            const int32_t ww = w % wpr;
            const int32_t r = w / wpr;
            const int32_t hl = r % Hl;
            const int32_t t = r / Hl;
            const uint64_t widx = ((base + t) * (uint64_t)H + (uint64_t)(rank * Hl + hl)) * (uint64_t)wpr + ww;
            dst[w] = splitmix64(widx + seedk);
        }
    }
}

}  // namespace

cudaError_t launch_xfer(bool gather, const XferDesc *desc, int64_t n, const XferGeom &g, void *kv, int32_t *table,
                        int ctas, int threads, int variant, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t M = n * g.two_l;
    if (variant == 1) {   // TMA bulk: one CTA per SM, kStages x piece bytes of smem ring
        const int32_t piece = (int32_t)std::min<int64_t>(g.chunk, 16384);
        if (ctas <= 0) ctas = 148;
        int64_t grid = std::min<int64_t>(ctas, M);
        const int64_t cpc = (M + grid - 1) / grid;
        grid = (M + cpc - 1) / cpc;
        const int64_t max_nb = cpc / g.two_l + 2;
        const size_t smem = (size_t)kStages * piece + kStages * sizeof(uint64_t) + (size_t)max_nb * sizeof(XferDesc);
        auto fn = gather ? k_xfer_bulk<true> : k_xfer_bulk<false>;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        fn<<<(unsigned)grid, 32, smem, s>>>(desc, n, g, static_cast<char *>(kv), table, cpc, piece);
        return cudaGetLastError();
    }
    if (threads <= 0 || threads > 256) threads = 256;
    if (ctas <= 0) ctas = 148 * 4;
    const int64_t nwarps = threads / 32;
    int64_t grid = std::min<int64_t>(ctas, (M + nwarps - 1) / nwarps);
    if (grid < 1) grid = 1;
    const int64_t cpc = (M + grid - 1) / grid;
    grid = (M + cpc - 1) / cpc;
    const int64_t max_nb = cpc / g.two_l + 2;
    const size_t smem = (size_t)max_nb * sizeof(XferDesc);
    if (smem > 48 * 1024) {
        auto fn = gather ? k_xfer<true> : k_xfer<false>;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (gather)
        k_xfer<true><<<(unsigned)grid, threads, smem, s>>>(desc, n, g, static_cast<char *>(kv), table, cpc);
    else
        k_xfer<false><<<(unsigned)grid, threads, smem, s>>>(desc, n, g, static_cast<char *>(kv), table, cpc);
    return cudaGetLastError();
}

cudaError_t launch_xfer_inline(bool gather, const XferDesc *host_desc, int32_t n, const XferGeom &g, void *kv,
                               int32_t *table, int ctas, int threads, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n > kMaxInlineDesc) return cudaErrorInvalidValue;
    InlineDescs d;
    for (int i = 0; i < n; ++i) d.d[i] = host_desc[i];
    const int64_t M = (int64_t)n * g.two_l;
    if (threads <= 0 || threads > 256) threads = 256;
    if (ctas <= 0) ctas = 148 * 4;
    const int64_t nwarps = threads / 32;
    int64_t grid = std::min<int64_t>(ctas, (M + nwarps - 1) / nwarps);
    if (grid < 1) grid = 1;
    const int64_t cpc = (M + grid - 1) / grid;
    grid = (M + cpc - 1) / cpc;
    if (gather)
        k_xfer_inl<true><<<(unsigned)grid, threads, 0, s>>>(d, n, g, static_cast<char *>(kv), table, cpc);
    else
        k_xfer_inl<false><<<(unsigned)grid, threads, 0, s>>>(d, n, g, static_cast<char *>(kv), table, cpc);
    return cudaGetLastError();
}

cudaError_t launch_fill(void *kv, int64_t n_pool, int32_t L, int32_t T, int32_t H, int32_t Hl, int32_t rank,
                        int32_t D, uint64_t seed, cudaStream_t s) {
    const int32_t wpr = D * 2 / 8;
    const int64_t n_chunks = (int64_t)L * 2 * n_pool;
    const uint64_t seedk = seed * 0xD1B54A32D192ED03ull;
    const int64_t grid = std::min<int64_t>(n_chunks, 148 * 16);
    k_fill<<<(unsigned)grid, 256, 0, s>>>(static_cast<uint64_t *>(kv), n_chunks, n_pool, T, H, Hl, rank, wpr, seedk);
    return cudaGetLastError();
}

}  // namespace tc
