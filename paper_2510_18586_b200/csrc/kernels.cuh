// Internal launch interface of the sm_100a kernels (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tc {

// One transfer descriptor per block (16 B).  `ext` is the device-visible address of the block's contiguous
// [L][2][C] image outside the pool: a mapped pinned host slot (DIRECT), a device staging slot (STAGED) or a caller
// buffer (device tier).  `tab` is the flat index of the block-table entry the fused epilogue rewrites
// (agent * row_stride + pos), or -1 for none.
struct XferDesc {
    int32_t blk;
    int32_t tab;
    uint64_t ext;
};
static_assert(sizeof(XferDesc) == 16, "XferDesc must be 16 bytes");

// Descriptors travel by value in the kernel parameters (<= 32 KiB of parameter space); larger batches are launched
// in pieces of at most kMaxInlineDesc blocks.
constexpr int kMaxInlineDesc = 2040;

struct XferGeom {
    int64_t n_pool;      // N
    int64_t chunk;       // C bytes (multiple of 16)
    int32_t two_l;       // 2L chunks per block
    unsigned long long *ts = nullptr;   // optional {first CTA start, last CTA end} in %globaltimer ns (tc_timing)
};

// gather: ext[i] + lk*C  <-  kv + (lk*N + blk_i)*C      (a3: offload; epilogue table[tab_i] = -1)
// scatter: kv + (lk*N + blk_i)*C  <-  ext[i] + lk*C     (a6: upload; epilogue table[tab_i] = blk_i)
// host_desc: n <= kMaxInlineDesc descriptors in host memory, copied into the launch's parameters.  ctas <= 0 selects
// the variant's default grid.  variant 0 = SIMT warp-per-chunk 16-byte copy; 1 = TMA bulk (cp.async.bulk) through
// an 8-stage shared-memory ring, one CTA per SM; 2 = SIMT tile split (4 KiB warp tiles spread evenly over all CTAs);
// 3 = TMA bulk, 4-stage ring, two CTAs per SM; 4 = SIMT 8 KiB tiles of 32-byte vectors (L2::256B; C % 32 == 0).
cudaError_t launch_xfer(bool gather, const XferDesc *host_desc, int32_t n, const XferGeom &g, void *kv,
                        int32_t *table, int ctas, int threads, int variant, cudaStream_t s);

// Table epilogue without a copy (COPY mode): table[tab_i] = gather ? -1 : blk_i for every descriptor with tab >= 0.
cudaError_t launch_table(bool gather, const XferDesc *host_desc, int64_t n, int32_t *table, cudaStream_t s);

// Synthetic content: word w of the unsharded [L][2][N][T][H][D] pool =
// splitmix64(w + seed * 0xD1B54A32D192ED03); this shard holds heads [rank*Hl, (rank+1)*Hl).
cudaError_t launch_fill(void *kv, int64_t n_pool, int32_t L, int32_t T, int32_t H, int32_t Hl, int32_t rank,
                        int32_t D, uint64_t seed, cudaStream_t s);

}  // namespace tc
