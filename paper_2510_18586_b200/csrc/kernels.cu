// sm_100a gather / scatter kernels of the Tokencake offload/upload hot path, and the synthetic-content fill kernel.
//
// Data movement only — no tensor cores (no contraction anywhere on this path).  A launch moves the
// 2L chunks (C contiguous bytes each, one per (layer, K|V)) of up to kMaxInlineDesc blocks between the paged pool
// [L][2][N][C] and each block's contiguous [L][2][C] image elsewhere (a mapped pinned host slot, a device staging
// slot or a caller buffer).  The warp / thread that moves byte 0 of a block also performs the fused block-table
// epilogue (P:649 location flag on offload, P:388 remap on upload).
//
// Descriptors travel BY VALUE in the kernel parameters (up to 32 KiB of parameter space, 2040 descriptors): a CTA
// reads its descriptors from the constant bank, so no launch reads host memory for its control data and no copy has
// to precede it.  (Measured on B200: CTAs fetching descriptors from a mapped pinned ring serialise at ~30 ns per CTA
// on the host link, which made wide grids slower than narrow ones; profiles/r01_tier_probe_v1.json.)
//
// Variants (same bytes, different engines; tc_set_launch_config):
//   0  SIMT, one warp per chunk (16-byte vectors, 8 in flight per lane)
//   1  TMA bulk, one elected thread per CTA streams 16 KiB pieces through an 8-stage shared-memory ring (1 CTA/SM)
//   2  SIMT, the launch's chunks cut into 4 KiB warp tiles split evenly over all CTAs
//   3  TMA bulk, 4-stage ring (2 CTAs/SM)
//   4  SIMT, 8 KiB warp tiles of 32-byte vectors with the L2::256B fetch hint (C % 32 == 0; else variant 2)
// Work is split over CTAs at piece/tile granularity (variants 1-3), so a small launch (the staged head/tail piece)
// still reaches every SM and a large one has no chunk-granular tail.
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "kernels.cuh"

namespace tc {
namespace {

constexpr int kUnroll = 8;
constexpr int kTileU = 8;
constexpr int64_t kTileBytes = kTileU * 512;   // one warp-iteration: 32 lanes x kTileU 16-byte vectors
constexpr int64_t kPieceMax = 16384;           // TMA bulk piece (bytes per cp.async.bulk)

// TMA ring bytes per CTA, overridable for tuning (TC_TMA_RING_KIB); 0 = by variant.
inline int64_t tma_ring_override() {
    static const int64_t v = [] {
        const char *e = std::getenv("TC_TMA_RING_KIB");
        return e ? std::atoll(e) * 1024 : 0ll;
    }();
    return v;
}

template <int kCap>
struct Descs {
    XferDesc d[kCap];
};

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

// Device-side launch timing (tc_timing): CTA 0's start (CTAs are dispatched in index order, so it is the first) and
// the latest CTA end on the %globaltimer clock (ns), so a kernel's duration excludes host launch latency.  Only CTA 0
// stamps the start: thousands of same-address atomics at launch would serialise at one L2 slice and delay the first
// loads by microseconds.  g.ts = {start, end}, pre-set to {UINT64_MAX, 0}; null = off.
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ts_begin(const XferGeom &g) {
    if (g.ts && blockIdx.x == 0) atomicMin(g.ts, now_ns());
}
__device__ __forceinline__ void ts_end(const XferGeom &g) {
    if (g.ts) atomicMax(g.ts + 1, now_ns());
}

// Byte address of offset `off` of chunk lk of descriptor d, in the pool and in the block's contiguous image.
struct Loc {
    char *pool, *ext;
};
__device__ __forceinline__ Loc locate(const XferDesc &d, int64_t lk, int64_t off, const XferGeom &g, char *kv) {
    return {kv + (lk * g.n_pool + d.blk) * g.chunk + off, reinterpret_cast<char *>(d.ext) + lk * g.chunk + off};
}

// ------------------------------------------------------------------------------------------------ variant 0
template <bool kGather>
__device__ __forceinline__ void chunk_body(const XferDesc *__restrict__ desc, int64_t n, const XferGeom &g,
                                           char *__restrict__ kv, int32_t *__restrict__ table, int64_t per_cta) {
    const int64_t M = n * g.two_l;
    const int64_t j0 = (int64_t)blockIdx.x * per_cta;
    if (j0 >= M) return;
    if (threadIdx.x == 0) ts_begin(g);
    const int64_t j1 = min(M, j0 + per_cta);
    const int lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int64_t nv = g.chunk >> 4;
    for (int64_t j = j0 + (threadIdx.x >> 5); j < j1; j += nwarps) {
        const int64_t i = j / g.two_l;
        const int64_t lk = j - i * g.two_l;
        const XferDesc d = desc[i];
        const Loc p = locate(d, lk, 0, g, kv);
        const int4 *src = reinterpret_cast<const int4 *>(kGather ? p.pool : p.ext);
        int4 *dst = reinterpret_cast<int4 *>(kGather ? p.ext : p.pool);
        int64_t v = lane;
        for (; v + 32 * (kUnroll - 1) < nv; v += 32 * kUnroll) {
            int4 r[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) r[u] = ld_stream(src + v + 32 * u);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) st_stream(dst + v + 32 * u, r[u]);
        }
        for (; v < nv; v += 32) st_stream(dst + v, ld_stream(src + v));
        if (lk == 0 && lane == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
    }
    if (g.ts) {
        __syncthreads();
        if (threadIdx.x == 0) ts_end(g);
    }
}

// ------------------------------------------------------------------------------------------------ variant 2
template <bool kGather>
__device__ __forceinline__ void tile_body(const XferDesc *__restrict__ desc, int64_t n, const XferGeom &g,
                                          char *__restrict__ kv, int32_t *__restrict__ table, int64_t per_cta) {
    const int64_t tpc = (g.chunk + kTileBytes - 1) / kTileBytes;   // tiles per chunk
    const int64_t tpb = tpc * g.two_l;                              // tiles per block
    const int64_t Mt = n * tpb;
    const int64_t t0 = (int64_t)blockIdx.x * per_cta;
    if (t0 >= Mt) return;
    if (threadIdx.x == 0) ts_begin(g);
    const int64_t t1 = min(Mt, t0 + per_cta);
    const int lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int64_t t = t0 + (threadIdx.x >> 5); t < t1; t += nwarps) {
        const int64_t i = t / tpb;
        const int64_t r = t - i * tpb;
        const int64_t lk = r / tpc;
        const int64_t off = (r - lk * tpc) * kTileBytes;
        const XferDesc d = desc[i];
        const Loc p = locate(d, lk, off, g, kv);
        const int4 *src = reinterpret_cast<const int4 *>(kGather ? p.pool : p.ext);
        int4 *dst = reinterpret_cast<int4 *>(kGather ? p.ext : p.pool);
        const int64_t nv = min(kTileBytes, g.chunk - off) >> 4;
        if (nv == kTileU * 32) {
            int4 v[kTileU];
#pragma unroll
            for (int u = 0; u < kTileU; ++u) v[u] = ld_stream(src + lane + 32 * u);
#pragma unroll
            for (int u = 0; u < kTileU; ++u) st_stream(dst + lane + 32 * u, v[u]);
        } else {
            for (int64_t v = lane; v < nv; v += 32) st_stream(dst + v, ld_stream(src + v));
        }
        if (r == 0 && lane == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
    }
    if (g.ts) {
        __syncthreads();
        if (threadIdx.x == 0) ts_end(g);
    }
}

// ------------------------------------------------------------------------------------------------ variant 4
// SIMT tile split like variant 2 with 32-byte vectors (LDG/STG .256) and the L2::256B fetch-size hint on the loads:
// a warp iteration moves 32 lanes x kTileU x 32 B = 8 KiB.  Meant for mapped host memory, where the size of each
// sysmem request may decide how many requests the link carries.  Needs C % 32 == 0 (else the launch uses variant 2).
struct V8 {
    uint32_t r[8];
};
__device__ __forceinline__ V8 ld_stream8(const V8 *p) {
    V8 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]),
                   "=r"(v.r[7])
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream8(V8 *p, const V8 &v) {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.r[0]),
                 "r"(v.r[1]), "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7])
                 : "memory");
}
constexpr int64_t kTile8Bytes = kTileU * 32 * 32;

template <bool kGather>
__device__ __forceinline__ void tile8_body(const XferDesc *__restrict__ desc, int64_t n, const XferGeom &g,
                                           char *__restrict__ kv, int32_t *__restrict__ table, int64_t per_cta) {
    const int64_t tpc = (g.chunk + kTile8Bytes - 1) / kTile8Bytes;
    const int64_t tpb = tpc * g.two_l;
    const int64_t Mt = n * tpb;
    const int64_t t0 = (int64_t)blockIdx.x * per_cta;
    if (t0 >= Mt) return;
    if (threadIdx.x == 0) ts_begin(g);
    const int64_t t1 = min(Mt, t0 + per_cta);
    const int lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int64_t t = t0 + (threadIdx.x >> 5); t < t1; t += nwarps) {
        const int64_t i = t / tpb;
        const int64_t r = t - i * tpb;
        const int64_t lk = r / tpc;
        const int64_t off = (r - lk * tpc) * kTile8Bytes;
        const XferDesc d = desc[i];
        const Loc p = locate(d, lk, off, g, kv);
        const V8 *src = reinterpret_cast<const V8 *>(kGather ? p.pool : p.ext);
        V8 *dst = reinterpret_cast<V8 *>(kGather ? p.ext : p.pool);
        const int64_t nv = min(kTile8Bytes, g.chunk - off) >> 5;
        if (nv == kTileU * 32) {
            V8 v[kTileU];
#pragma unroll
            for (int u = 0; u < kTileU; ++u) v[u] = ld_stream8(src + lane + 32 * u);
#pragma unroll
            for (int u = 0; u < kTileU; ++u) st_stream8(dst + lane + 32 * u, v[u]);
        } else {
            for (int64_t v = lane; v < nv; v += 32) st_stream8(dst + v, ld_stream8(src + v));
        }
        if (r == 0 && lane == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
    }
    if (g.ts) {
        __syncthreads();
        if (threadIdx.x == 0) ts_end(g);
    }
}

// ------------------------------------------------------------------------------------------------ variants 1, 3
// One elected thread per CTA streams its piece range through a kStages-deep shared-memory ring with the TMA bulk-copy
// engine: cp.async.bulk global->shared (mbarrier complete_tx), then cp.async.bulk shared->global (bulk_group).  A
// stage is refilled as soon as the bulk store that drains it has finished READING shared memory (wait_group.read), so
// kStages loads stay in flight.  Pieces go to or from mapped host memory or HBM alike.
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
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Position of a piece inside the launch: block i, chunk lk of the block, piece q of the chunk.  Advanced one piece at
// a time, so the issuing thread does no 64-bit division in its loop.
struct Cursor {
    int64_t i;
    int32_t lk, q;
    __device__ __forceinline__ void init(int64_t k, int32_t ppc, int32_t two_l) {
        const int64_t ppb = (int64_t)ppc * two_l;
        i = k / ppb;
        const int32_t r = (int32_t)(k - i * ppb);
        lk = r / ppc;
        q = r - lk * ppc;
    }
    __device__ __forceinline__ void next(int32_t ppc, int32_t two_l) {
        if (++q == ppc) {
            q = 0;
            if (++lk == two_l) {
                lk = 0;
                ++i;
            }
        }
    }
};

constexpr int kMaxStages = 32;

template <bool kGather>
__device__ __forceinline__ void bulk_body(const XferDesc *__restrict__ desc, int64_t n, const XferGeom &g,
                                          char *__restrict__ kv, int32_t *__restrict__ table, int64_t per_cta,
                                          int32_t piece, int32_t stages, unsigned char *smem) {
    const int32_t ppc = (int32_t)((g.chunk + piece - 1) / piece);   // pieces per chunk
    const int64_t K = n * ppc * g.two_l;
    const int64_t k0 = (int64_t)blockIdx.x * per_cta;
    if (k0 >= K || threadIdx.x != 0) return;
    const int64_t total = min(K, k0 + per_cta) - k0;
    unsigned char *ring = smem;                                                      // stages x piece
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)stages * piece);  // stages mbarriers
    for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ts_begin(g);
    Cursor ld, st;
    ld.init(k0, ppc, g.two_l);
    st = ld;
    int sl = 0, ss = 0;
    uint32_t phase = 0;
    int64_t issued = 0;
    // load of the next piece into stage sl; the load of a block's first piece carries the table epilogue
    auto issue_load = [&]() {
        const XferDesc d = desc[ld.i];
        const int64_t off = (int64_t)ld.q * piece;
        const Loc p = locate(d, ld.lk, off, g, kv);
        const uint32_t bytes = (uint32_t)min((int64_t)piece, g.chunk - off);
        if (ld.lk == 0 && ld.q == 0 && d.tab >= 0) table[d.tab] = kGather ? -1 : d.blk;
        mbar_expect_tx(&bars[sl], bytes);
        bulk_load(ring + (size_t)sl * piece, kGather ? p.pool : p.ext, bytes, &bars[sl]);
        ld.next(ppc, g.two_l);
        if (++sl == stages) sl = 0;
        ++issued;
    };
    while (issued < total && issued < stages) issue_load();
    for (int64_t q = 0; q < total; ++q) {
        mbar_wait(&bars[ss], phase);
        const XferDesc d = desc[st.i];
        const int64_t off = (int64_t)st.q * piece;
        const Loc p = locate(d, st.lk, off, g, kv);
        bulk_store(kGather ? p.ext : p.pool, ring + (size_t)ss * piece, (uint32_t)min((int64_t)piece, g.chunk - off));
        bulk_commit();
        st.next(ppc, g.two_l);
        if (q >= 1 && issued < total) {   // refill the stage the previous store drained, once it has read smem
            bulk_wait_read1();
            issue_load();
        }
        if (++ss == stages) {
            ss = 0;
            phase ^= 1;
        }
    }
    bulk_wait_all();
    ts_end(g);
}

// ------------------------------------------------------------------------------------------------ kernels
template <bool kGather, int kCap>
__global__ void __launch_bounds__(256) k_xfer_chunk(const __grid_constant__ Descs<kCap> dd, int32_t n, XferGeom g,
                                                    char *__restrict__ kv, int32_t *__restrict__ table,
                                                    int64_t per_cta) {
    chunk_body<kGather>(dd.d, n, g, kv, table, per_cta);
}

template <bool kGather, int kCap>
__global__ void __launch_bounds__(256) k_xfer_tile(const __grid_constant__ Descs<kCap> dd, int32_t n, XferGeom g,
                                                   char *__restrict__ kv, int32_t *__restrict__ table,
                                                   int64_t per_cta) {
    tile_body<kGather>(dd.d, n, g, kv, table, per_cta);
}

template <bool kGather, int kCap>
__global__ void __launch_bounds__(256) k_xfer_tile8(const __grid_constant__ Descs<kCap> dd, int32_t n, XferGeom g,
                                                    char *__restrict__ kv, int32_t *__restrict__ table,
                                                    int64_t per_cta) {
    tile8_body<kGather>(dd.d, n, g, kv, table, per_cta);
}

template <bool kGather, int kCap>
__global__ void __launch_bounds__(32) k_xfer_bulk(const __grid_constant__ Descs<kCap> dd, int32_t n, XferGeom g,
                                                  char *__restrict__ kv, int32_t *__restrict__ table,
                                                  int64_t per_cta, int32_t piece, int32_t stages) {
    extern __shared__ __align__(128) unsigned char smem[];
    bulk_body<kGather>(dd.d, n, g, kv, table, per_cta, piece, stages, smem);
}

// Even split of `units` work units over at most `ctas` CTAs (each >= `min_per_cta` units): {grid, units per CTA}.
inline void split(int64_t units, int64_t ctas, int64_t min_per_cta, int64_t *grid, int64_t *per_cta) {
    const int64_t gsz = std::max<int64_t>(1, std::min<int64_t>(ctas, (units + min_per_cta - 1) / min_per_cta));
    *per_cta = (units + gsz - 1) / gsz;
    *grid = (units + *per_cta - 1) / *per_cta;
}

template <int kCap>
cudaError_t launch_cap(bool gather, const XferDesc *host_desc, int32_t n, const XferGeom &g, char *kv,
                       int32_t *table, int ctas, int threads, int variant, cudaStream_t s) {
    Descs<kCap> dd;
    std::copy(host_desc, host_desc + n, dd.d);
    int64_t grid = 0, per = 0;
    if (variant == 1 || variant == 3) {
        // ring bytes per CTA: 128 KiB, one CTA per SM (1) / 96 KiB, two resident per SM (3).  stages = ring / piece,
        // so small chunks (C5's 4 KiB) keep as many bytes in flight as large ones.  Variant 3's default grid follows
        // the launch size: ~128 KiB per CTA, between 2 and 15 CTAs per SM — several waves of short CTAs let the block
        // scheduler even out per-channel speed differences (profiles/r01_tier_probe_grid_v4.log: 0.95-1.0 of the HBM
        // copy peak from 100 MiB up, C2 and C5); up to 4 waves the grid is rounded to whole waves of 296 CTAs (two per
        // SM), so a launch never ends on a partial wave: 32 MiB runs as one wave instead of 1.5 waves of 444 (0.88-0.92
        // vs 0.81-0.84 of the copy peak), 4-16 MiB up to 30 % shorter, 47 MiB without its 1.3-wave tail
        // (profiles/r02_tier_probe_c{2,5}_*.json).
        const int32_t piece = (int32_t)std::min<int64_t>(g.chunk, kPieceMax);
        const int64_t K = (int64_t)n * g.two_l * ((g.chunk + piece - 1) / piece);
        const int64_t ring = tma_ring_override() > 0 ? tma_ring_override() : (variant == 1 ? 128 << 10 : 96 << 10);
        const int32_t stages = (int32_t)std::max<int64_t>(2, std::min<int64_t>(kMaxStages, ring / piece));
        int64_t want = ctas;
        if (want <= 0) {
            const int64_t bytes = (int64_t)n * g.two_l * g.chunk;
            want = bytes >> 17;                      // ~128 KiB per CTA
            if (variant == 1) {
                want = 148;
            } else if (want <= 1184) {               // up to 4 waves: whole waves of 296 (2 per SM), no partial one
                want = std::max<int64_t>(1, (want + 148) / 296) * 296;
            } else {
                want = std::min<int64_t>(2220, want);
            }
        }
        split(K, want, 1, &grid, &per);
        const size_t smem = (size_t)stages * piece + stages * sizeof(uint64_t);
        auto fn = gather ? k_xfer_bulk<true, kCap> : k_xfer_bulk<false, kCap>;
        // the opt-in dynamic shared memory is raised once per kernel (and device) to the largest size seen: a
        // cudaFuncSetAttribute on every launch sat on the host's launch path (tens of µs per launch).  Atomic: pools
        // on several host threads may launch at once; a racing raise just sets the attribute twice (idempotent).
        static std::atomic<size_t> smem_set[2][64] = {};
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
        std::atomic<size_t> &done = smem_set[gather ? 1 : 0][dev];
        size_t seen = done.load(std::memory_order_acquire);
        if (smem > seen) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            while (seen < smem && !done.compare_exchange_weak(seen, smem, std::memory_order_acq_rel)) {
            }
        }
        fn<<<(unsigned)grid, 32, smem, s>>>(dd, n, g, kv, table, per, piece, stages);
        return cudaGetLastError();
    }
    if (threads <= 0 || threads > 256) threads = 256;
    const int64_t nwarps = threads / 32;
    if (variant == 4 && g.chunk % 32 == 0) {
        const int64_t Mt = (int64_t)n * g.two_l * ((g.chunk + kTile8Bytes - 1) / kTile8Bytes);
        split(Mt, ctas > 0 ? ctas : 148 * 4, nwarps, &grid, &per);
        if (gather)
            k_xfer_tile8<true, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
        else
            k_xfer_tile8<false, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
        return cudaGetLastError();
    }
    if (variant == 4) variant = 2;                   // C % 32 != 0: 16-byte tiles
    if (variant == 2) {
        const int64_t Mt = (int64_t)n * g.two_l * ((g.chunk + kTileBytes - 1) / kTileBytes);
        split(Mt, ctas > 0 ? ctas : 148 * 4, nwarps, &grid, &per);
        if (gather)
            k_xfer_tile<true, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
        else
            k_xfer_tile<false, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
        return cudaGetLastError();
    }
    split((int64_t)n * g.two_l, ctas > 0 ? ctas : 148 * 4, nwarps, &grid, &per);
    if (gather)
        k_xfer_chunk<true, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
    else
        k_xfer_chunk<false, kCap><<<(unsigned)grid, threads, 0, s>>>(dd, n, g, kv, table, per);
    return cudaGetLastError();
}

// Table epilogue alone (COPY mode, where the copy engine moves the bytes): table[tab_i] = -1 (offload) / blk_i.
template <int kCap>
__global__ void k_table(const __grid_constant__ Descs<kCap> dd, int32_t n, bool gather, int32_t *__restrict__ table) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (dd.d[i].tab >= 0) table[dd.d[i].tab] = gather ? -1 : dd.d[i].blk;
}

template <int kCap>
cudaError_t launch_table_cap(bool gather, const XferDesc *host_desc, int32_t n, int32_t *table, cudaStream_t s) {
    Descs<kCap> dd;
    std::copy(host_desc, host_desc + n, dd.d);
    k_table<kCap><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dd, n, gather, table);
    return cudaGetLastError();
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

cudaError_t launch_xfer(bool gather, const XferDesc *host_desc, int32_t n, const XferGeom &g, void *kv,
                        int32_t *table, int ctas, int threads, int variant, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n > kMaxInlineDesc || variant < 0 || variant > 4) return cudaErrorInvalidValue;
    char *k = static_cast<char *>(kv);
    if (n <= 64) return launch_cap<64>(gather, host_desc, n, g, k, table, ctas, threads, variant, s);
    if (n <= 256) return launch_cap<256>(gather, host_desc, n, g, k, table, ctas, threads, variant, s);
    return launch_cap<kMaxInlineDesc>(gather, host_desc, n, g, k, table, ctas, threads, variant, s);
}

cudaError_t launch_table(bool gather, const XferDesc *host_desc, int64_t n, int32_t *table, cudaStream_t s) {
    for (int64_t a = 0; a < n; a += kMaxInlineDesc) {
        const int32_t m = (int32_t)std::min<int64_t>(kMaxInlineDesc, n - a);
        cudaError_t e = m <= 256 ? launch_table_cap<256>(gather, host_desc + a, m, table, s)
                                 : launch_table_cap<kMaxInlineDesc>(gather, host_desc + a, m, table, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
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
