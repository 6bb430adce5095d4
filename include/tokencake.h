/*
 * tokencake.h — C ABI of the B200-native Tokencake Time-Scheduler hot path (arXiv 2510.18586).
 *
 * What it does (§4 "The Time Scheduler", and §Implementation): while an agent stalls on
 * a function call, its paged KV-cache blocks — non-contiguous (block, layer, K|V) chunks of a layer-major pool — are
 * gathered into pinned host memory taken from an internal free list ("CPU Block Buffering"); the source
 * GPU blocks become "pending free" and return to the pool only after the transfer completes.  Before the call
 * returns they are scattered back into freshly allocated GPU blocks and the agent's block table is remapped
 * (P:388).  Allocation honours the Space Scheduler's per-class reservations: a shared pool plus a
 * reserved pool per critical agent class (Alg. 2 line 15 reserve_num[agent_type]).
 *
 * Conventions:
 *  - One pool per (process, CUDA device).  Not thread-safe: a single writer, as S:204-205.
 *  - Ownership: the caller owns every array it passes; inputs are copied before return; outputs are written only on
 *    TC_OK.  Handles, pinned host slots, streams, events and (unless supplied externally) device memory are owned by
 *    the library and released by tc_pool_destroy.
 *  - Errors: strong guarantee — a non-OK status other than TC_E_CUDA leaves every piece of state unchanged
 *    ("pool unchanged").  TC_E_NOHOST (offload refused) and TC_E_NOBLOCKS (upload "stalls",
 *    S:178; the handle stays valid) are recoverable: retry after sync / free / re-quota.  TC_E_OOM from a host
 *    allocation is recoverable when it happens while a call is validated (nothing changed); the rare one after part
 *    of a batch's GPU work was enqueued poisons the pool like TC_E_CUDA.  TC_E_CUDA is sticky: the pool refuses
 *    further work and tc_last_error() says why.
 *  - Asynchrony: tc_offload / tc_upload return once the work is enqueued on the library's copy streams.  Logical
 *    state (block tables, counters) changes at call time; device/host bytes are valid after tc_wait / tc_stream_wait
 *    / tc_sync.  Freed device blocks and released host slots are reusable only after a retirement point — tc_sync
 *    (reading A8), tc_retire (A8') or tc_retire_lag (A8''), each of which waits for exactly the transfers it
 *    retires — so every id is a pure function of the call sequence, never of copy timing.
 *  - Layouts: KV pool [L][2][N][T][H/G][D] of 16-bit words (layer-major; chunk (block, layer, K|V) = C contiguous
 *    bytes, C = T*(H/G)*D*2; reading A3).  A host slot holds one block shard [L][2][C] = B = 2*L*C bytes (A4).
 *    Device block table int32[max_agents][max_blocks_per_agent], -1 = on host (A17).
 *  - Payload is opaque 16-bit words: never converted; NaN payloads, -0 and denormals survive (A14).
 */
#ifndef TOKENCAKE_H
#define TOKENCAKE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_pool tc_pool;      /* opaque, library-owned */
typedef uint64_t tc_handle;          /* 0 = none; issued 1, 2, 3, ... in call order */

typedef enum { TC_FP16 = 0, TC_BF16 = 1 } tc_dtype;

typedef enum {
    TC_OK = 0,
    TC_E_INVAL = -1,     /* bad argument: n < 1, duplicate ids, id not an on-GPU block of the agent, unknown agent /
                            class, sum of reservations > N, table row capacity exceeded (A15, A5, A9, A22) */
    TC_E_NOBLOCKS = -2,  /* not enough free device blocks under the partition rule; nothing changed */
    TC_E_NOHOST = -3,    /* host block buffer exhausted; offload refused, nothing changed */
    TC_E_HANDLE = -4,    /* unknown handle, or already uploaded */
    TC_E_BUSY = -5,      /* agent_free while the agent has offloaded blocks / query: transfer still running */
    TC_E_CUDA = -6,      /* CUDA error (sticky); see tc_last_error */
    TC_E_OOM = -7,       /* device / pinned-host allocation failed at create time, or a host allocation failed */
    TC_E_NODEV = -8      /* operation needs KV storage but the pool is metadata-only (device = -1) */
} tc_status;

typedef enum {
    TC_XFER_AUTO = 0,    /* per direction: STAGED, the path measured fastest for the cycle on B200 (re-measured on
                            this box by tc_calibrate), except that a batch up to the small-batch crossover (2 MiB
                            until tc_calibrate measures it per direction) takes DIRECT (one launch, lower latency;
                            DESIGN.md §6) */
    TC_XFER_DIRECT = 1,  /* one SM kernel reads/writes mapped pinned host memory over the host link */
    TC_XFER_STAGED = 2,  /* TMA gather/scatter to a device staging buffer + one copy-engine DMA per contiguous run
                            of host slots */
    TC_XFER_COPY = 3     /* the copy engine moves each block as one strided DMA (2L rows of C bytes, row pitch N*C in
                            the pool) straight between the pool and its pinned slot; a small kernel rewrites the
                            block table (offload: before the DMA; upload: after it) */
} tc_xfer_mode;

typedef struct tc_pool_desc {
    int32_t layers, kv_heads, head_dim, block_tokens;
    tc_dtype dtype;
    int64_t n_blocks;            /* N: blocks in this GPU's pool */
    int32_t device;              /* CUDA ordinal; -1 = metadata-only pool: allocator, tables and handles without KV
                                    storage or transfers (host-logic testing; data ops return TC_E_NODEV) */
    int32_t shard_rank, shard_world;   /* head shard: local heads = kv_heads / shard_world (must divide), A19 */
    int64_t host_slots;          /* S: pinned host block-shard slots; 0 -> ceil(0.18 * N) */
    int32_t n_classes;           /* agent classes, 1..64; 0 -> 8 */
    int32_t max_agents;          /* block-table rows; 0 -> 1024 */
    int32_t max_blocks_per_agent;/* block-table row capacity; 0 -> 4096 */
    void *kv_dev;                /* optional external device buffer (e.g. torch-allocated) >= L*2*N*C bytes,
                                    16-byte aligned; NULL -> library cudaMalloc */
    int32_t *table_dev;          /* optional external device int32[max_agents][max_blocks_per_agent]; NULL -> own */
    int32_t xfer_d2h, xfer_h2d;  /* tc_xfer_mode per direction */
    int64_t staging_bytes;       /* device staging buffer per direction for STAGED mode (allocated on first use); a
                                    larger batch runs double-buffered halves; 0 -> 1 GiB */
    int64_t desc_bytes;          /* pinned ring for block-table pushes (tc_alloc growth); 0 -> 16 MiB */
    int32_t unbuffered;          /* ABLATION ONLY (Fig. 11): no CPU block buffer — each offload
                                    cudaHostAlloc's its own pinned memory, freed (cudaFreeHost) when its upload
                                    retires; the bursty host allocation pattern of P:470-479.  0 = normal. */
    /* NEXT-2 peer tier ("a neighboring GPU's memory over high-speed interconnects like NVLink as a
       faster offload target than CPU RAM"; reading C1).  peer_slots > 0 block-shard slots are allocated
       in peer_device's HBM (peer access enabled; peer_device == device is allowed: an HBM-resident tier).  An
       offload goes whole to the peer tier when its free list holds all the blocks, else whole to the host buffer,
       else TC_E_NOHOST.  Peer slots are moved by the device-side gather/scatter kernel writing/reading the peer's
       memory directly (launch path 3).  Incompatible with `unbuffered` (TC_E_INVAL).  Defaults: -1 / 0 = none. */
    int32_t peer_device;
    int64_t peer_slots;
} tc_pool_desc;

typedef struct tc_stats_t {
    int64_t n_blocks, free_blocks, alloc_blocks, pending_blocks;
    int64_t host_slots, host_free, host_used, host_released;
    int64_t chunk_bytes, block_bytes;
    int32_t n_classes, n_agents;
    int64_t reserved[64], claimed[64];
    int64_t live_handles;
    int64_t kernel_launches, memcpy_calls;     /* cumulative, this pool */
    int64_t bytes_d2h, bytes_h2d;              /* cumulative KV payload bytes enqueued */
    int32_t xfer_d2h, xfer_h2d;                /* effective modes (AUTO resolved) */
    int64_t reserved_blocks;                   /* claimed by gradual reservations, not yet uploaded into */
    int64_t peer_slots, peer_free, peer_used;  /* NEXT-2 peer tier (0 without one) */
} tc_stats_t;

/* ---- pool lifecycle ------------------------------------------------------------------------------------------ */
/* Fill *d with defaults for the given geometry (device = current CUDA device). */
void tc_pool_desc_init(tc_pool_desc *d, int32_t layers, int32_t kv_heads, int32_t head_dim, int32_t block_tokens,
                       tc_dtype dtype, int64_t n_blocks);
/* P:601 paged pool (vLLM PagedAttention): N blocks of T tokens x all layers x K,V x local heads x head_dim. */
tc_status tc_pool_create(int32_t layers, int32_t kv_heads, int32_t head_dim, int32_t block_tokens, tc_dtype dtype,
                         int64_t n_blocks, tc_pool **out);
tc_status tc_pool_create_ex(const tc_pool_desc *d, tc_pool **out);
void tc_pool_destroy(tc_pool *p);
/* Device KV base pointer (layout above) and chunk bytes C. */
tc_status tc_pool_kv(tc_pool *p, void **kv_dev, int64_t *chunk_bytes);
/* The engine's compute (decode) stream.  Every later offload waits GPU-side for the work queued on it at the call, so
   an agent's last decode writes are in the offloaded image (S:283 resume safety, P:645-648 cycle order), and
   block-table pushes (tc_alloc) go on it.  NULL = none (pushes go on the offload stream).  The caller keeps the
   stream alive while it is set. */
tc_status tc_set_compute_stream(tc_pool *p, void *cuda_stream);
/* The library's copy streams (upload = high priority), for event timing / dependencies by the caller. */
tc_status tc_streams(tc_pool *p, void **upload_stream, void **offload_stream);
/* Override the transfer mode per direction (tc_xfer_mode) for subsequent calls. */
tc_status tc_set_xfer_mode(tc_pool *p, int32_t d2h, int32_t h2d);
/* Measure, on this box, which path AUTO should take (north_star: direct mapped-host writes "chosen against a
   device-staging path plus cudaMemcpyAsync according to the measured bandwidth"): a full cycle — an offload of
   probe_bytes (gather) and an upload of probe_bytes (scatter) running concurrently — is timed (best of 3) for each of
   the four {DIRECT, STAGED} x {DIRECT, STAGED} combinations; AUTO directions then take the fastest combination.
   Uses pool blocks [0, 2k) and 2k free host slots (k = probe_bytes / B, shrunk to what is free; TC_E_NOHOST if not
   even 1 + 1 fit): the gathered blocks are only read and the scattered ones receive their own bytes back, so the pool's
   contents are unchanged — but the caller must not run kernels on the pool meanwhile.  Blocking.
   gbs[i] = 2 * probe bytes / cycle time for combination i = 2 * (d2h is STAGED) + (h2d is STAGED).  Then, per
   direction alone, batches of 1, 2, 4, ... (<= 64) blocks are timed DIRECT vs STAGED: AUTO sends batches up to the
   largest size where DIRECT was never slower (direct_max_bytes[dir]; 0 = never) through the DIRECT kernel. */
typedef struct tc_calibration_t {
    int32_t d2h, h2d;          /* the chosen modes (what AUTO directions now use) */
    int64_t probe_bytes;       /* bytes per direction actually probed */
    double gbs[4];
    int64_t direct_max_bytes[2];   /* [0] offload (D2H), [1] upload (H2D): AUTO's small-batch DIRECT crossover */
} tc_calibration_t;
tc_status tc_calibrate(tc_pool *p, int64_t probe_bytes, tc_calibration_t *out);
/* Launch configuration of one kernel path: path 0 = direct D2H gather, 1 = direct H2D scatter, 2 = device-side
   gather/scatter (staged mode and device tier), 3 = peer-tier gather/scatter (NEXT-2).  ctas <= 0 -> default grid;
   threads in {32..256} (SIMT variants);
   variant 0 = SIMT warp-per-chunk 16-byte copies, 1 = TMA bulk copies (cp.async.bulk through an 8-stage
   shared-memory ring, one elected thread per CTA, one CTA per SM), 2 = SIMT tile split (4 KiB warp tiles spread
   evenly over all CTAs), 3 = TMA bulk with a 4-stage ring (two CTAs per SM), 4 = SIMT tiles of 32-byte vectors with
   the L2::256B fetch hint (C % 32 == 0, else as 2).  Other values -> TC_E_INVAL.
   Results are identical for every setting; only speed differs.  Defaults (at create; TC_CTAS_* / TC_VARIANT_*
   override): variant 3 on every path; 32 CTAs for path 0, 74 for path 1 (a DIRECT kernel occupies its SMs for the
   whole link transfer, so it gets a small fixed grid that leaves the other direction room), the size-adaptive grid
   (ctas = 0) for paths 2 and 3.  ctas <= 0 here restores the variant's size-adaptive grid. */
tc_status tc_set_launch_config(tc_pool *p, int32_t path, int32_t ctas, int32_t threads, int32_t variant);
/* Synthetic content: every 8-byte word of the unsharded pool = splitmix64(widx + seed*0xD1B54A32D192ED03), widx its
   index in [L][2][N][T][H][D]; this rank writes its head shard.  Tests/bench only. */
tc_status tc_fill_kv(tc_pool *p, uint64_t seed);

/* ---- Space-Scheduler partition + agents (a1, a5) ------------------------------------------------------------ */
/* reserve_num[agent_class] = n_blocks.  Counts, not address ranges (A9).  Requires sum over classes <= N.
   claimed is untouched: a shrink below claimed is lazy. */
tc_status tc_partition_reserve(tc_pool *p, int32_t agent_class, int64_t n_blocks);
tc_status tc_agent_add(tc_pool *p, int32_t agent, int32_t agent_class);
/* Decode growth: append n blocks to the agent's table; ids = lowest free first (A7), reservation first then shared
   headroom = free - sum of unclaimed reservations.  out_ids[n] receives them. */
tc_status tc_alloc(tc_pool *p, int32_t agent, int64_t n, int32_t *out_ids);
/* Release all the agent's on-GPU blocks (reservation-first return).  TC_E_BUSY while it has offloaded
   blocks.  The caller guarantees no queued compute still uses them. */
tc_status tc_agent_free(tc_pool *p, int32_t agent);

/* ---- the hot path (a2-a8) ----------------------------------------------------------------------------------- */
/* a2+a3: offload block_ids[0..n) (on-GPU blocks exclusively owned by the agent) to pinned host slots from the
   CPU block buffer; gather all 2L chunks of each block in one kernel launch; table entries -> -1 (device table
   written by the kernel epilogue); source blocks PENDING until a retirement point that covers this call — tc_sync,
   tc_retire, tc_retire_lag (A8, A8', A8'').  *out = new handle. */
tc_status tc_offload(tc_pool *p, int32_t agent, const int32_t *block_ids, int64_t n, tc_handle *out);
/* a5+a6: allocate n new blocks (rule of tc_alloc) and scatter the handle's host copy into them; the kernel's fused
   epilogue writes table[agent][pos_i] = out_new_ids[i] (new_ids[i] replaces block_ids[i], A6).  Upload waits
   (GPU-side) for the handle's offload (A13).  NOBLOCKS: nothing changes, the handle stays valid. */
tc_status tc_upload(tc_pool *p, tc_handle h, int32_t *out_new_ids);
/* a8: one scheduling cycle's offloads as ONE launch.  Agent k offloads block_ids[offsets[k]..offsets[k+1]).
   All-or-nothing. out_handles[n_agents]. */
tc_status tc_offload_batch(tc_pool *p, int32_t n_agents, const int32_t *agents, const int64_t *offsets,
                           const int32_t *block_ids, tc_handle *out_handles);
/* a8: one cycle's uploads as ONE launch; offsets[n_handles+1] must match each handle's block count (see
   tc_handle_info).  Sequential-composition semantics, all-or-nothing.  out_new_ids[offsets[n_handles]]. */
tc_status tc_upload_batch(tc_pool *p, int32_t n_handles, const tc_handle *hs, const int64_t *offsets,
                          int32_t *out_new_ids);
/* a8: one whole scheduling cycle in one call — the cycle's uploads (tc_upload_batch arguments) then its offloads
   (tc_offload_batch arguments).  Everything is validated before anything changes: all-or-nothing, the
   uploads' status reported first.  Offloads are validated against the pre-cycle state, so they cannot name blocks
   this cycle's uploads allocate (TC_E_INVAL; reading B5).  The two directions are enqueued interleaved so
   both host-link directions start as early as possible.  n_handles or n_agents may be 0 (that half is skipped). */
tc_status tc_cycle(tc_pool *p, int32_t n_handles, const tc_handle *hs, const int64_t *up_offsets,
                   int32_t *out_new_ids, int32_t n_agents, const int32_t *agents, const int64_t *off_offsets,
                   const int32_t *block_ids, tc_handle *out_handles);

/* ---- NEXT-1: Gradual GPU Block Reservation ------------------------------------------ */
/* Plan to claim an offloaded handle's n destination blocks over `cycles` scheduling ticks: chunk t of a near-equal,
   largest-first split (100/4 -> 25,25,25,25; 10/3 -> 4,3,3).  TC_E_INVAL if cycles < 1 or one is already active. */
tc_status tc_reserve_begin(tc_pool *p, tc_handle h, int32_t cycles);
/* One scheduling tick: every handle with an active plan (issue order) claims, under its class's partition rule,
   up to its cumulative target; a shortfall carries to the next tick.  Claimed blocks are RESERVED: not free,
   not owned, no data.  tc_upload / tc_upload_batch use them first (claim order), then allocate the remainder. */
tc_status tc_reserve_tick(tc_pool *p);
/* Return a handle's reserved blocks to the pool at once (reservation-first return). */
tc_status tc_reserve_cancel(tc_pool *p, tc_handle h);
tc_status tc_reserve_info(tc_pool *p, tc_handle h, int64_t *reserved, int64_t *total);   /* readiness */

/* Completion of a handle's latest transfer (a4 / a7; "after the transfer is complete", "never resumes
   decode while any of its blocks are host-resident or in flight").  tc_query: TC_OK if it has completed, TC_E_BUSY
   if not, TC_E_HANDLE if the handle is unknown (or forgotten, reading B3).  tc_wait: host-blocking wait.
   tc_stream_wait: makes `cuda_stream` wait GPU-side (no host block) — the engine's decode of an uploaded agent is
   enqueued after it and reads the scattered blocks and remapped table.  No state changes.  In a staged batch that
   runs as several pieces, each handle completes with the piece holding its last block, not with the whole batch,
   and each piece waits only for the handles / agents it holds (TC_FINE_DEPS=0: batch granularity). */
tc_status tc_query(tc_pool *p, tc_handle h);
tc_status tc_wait(tc_pool *p, tc_handle h);                        /* host-blocking */
tc_status tc_stream_wait(tc_pool *p, tc_handle h, void *cuda_stream); /* GPU-side dependency, no host block */
/* Drain both copy streams; retire PENDING device blocks (FREE, claimed -= min(n, claimed)) in issue order, then
   return released host slots to the free list.  Uploaded handles are forgotten.  A retirement point. */
tc_status tc_sync(tc_pool *p);
/* Retire without draining (reading A8'; "only returned to the memory pool after the transfer is
   complete", P:411 asynchronous transfers): waits for, and retires exactly as tc_sync would, only the work enqueued
   before the previous retirement point (tc_sync or tc_retire); work enqueued since keeps running and stays pending.
   A serving loop calling tc_retire once per scheduling cycle returns last cycle's blocks and slots while this
   cycle's transfers stream on.  Ids stay a pure function of the call sequence.  A retirement point. */
tc_status tc_retire(tc_pool *p);
/* Retire with a lag (reading A8''; same passages): as tc_retire, but against the lag-th previous
   retirement point — waits for and retires only the work enqueued before it, so the transfers of the last `lag`
   scheduling cycles keep streaming while the caller enqueues the next one (a deeper asynchronous loop when one
   cycle's uploads and offloads are unbalanced).  lag = 1 is tc_retire.  TC_E_INVAL for lag < 1 (no change, no new
   retirement point).  Ids stay a pure function of the call sequence.  A retirement point. */
tc_status tc_retire_lag(tc_pool *p, int32_t lag);

/* ---- queries ------------------------------------------------------------------------------------------------- */
/* The agent's block table (host mirror): out[pos] = device block id, -1 = host-resident (the location flag of
   P:649; reading A17); the remap of P:388 / P:646 is visible here at call time.  *n_out = the row length; at most
   cap entries are written; out == NULL only queries the length (TC_E_INVAL if cap < the row length or the agent
   is unknown). */
tc_status tc_block_table(tc_pool *p, int32_t agent, int32_t *out, int64_t cap, int64_t *n_out); /* -1 = on host */
/* The device copy of every table, int32[max_agents][row_stride], rewritten by the transfer kernels' epilogues in
   stream order (the fused remap); library-owned unless supplied at create. */
tc_status tc_block_table_dev(tc_pool *p, int32_t **dev_table, int64_t *row_stride);
/* agent, block count, state (1 = offloaded, 2 = uploaded) of a live handle */
tc_status tc_handle_info(tc_pool *p, tc_handle h, int32_t *agent, int64_t *n, int32_t *state);
/* Host pointer to the pinned copy of block i of an offloaded handle, layout [L][2][C] (valid after tc_wait). */
tc_status tc_handle_host(tc_pool *p, tc_handle h, int64_t i, const void **host_ptr);
/* Copy block i's image ([L][2][C], B bytes) of an offloaded handle — from its host slot or its peer-tier slot — into
   the caller's host buffer `dst` (blocking; waits for the handle's transfer).  TC_E_HANDLE if h is not offloaded,
   TC_E_INVAL for a bad i or dst, TC_E_NODEV on a metadata-only pool.  *tier (optional) = 0 host, 1 peer. */
tc_status tc_handle_read(tc_pool *p, tc_handle h, int64_t i, void *dst, int32_t *tier);
/* Allocator and transfer counters (S:113-115 conservation terms: free + alloc + pending (+ reserved) = N, host
   free + used + released = S; per-class reserved / claimed of P:519-521).  Read-only. */
tc_status tc_stats(tc_pool *p, tc_stats_t *s);
/* Per-launch device timing (CUDA events recorded on the launching stream around every kernel / memcpy run).
   Spans complete at tc_sync, where their durations are accumulated.  Index (TC_NKINDS): 0 staged-mode device-side
   gather kernels (offload), 1 staged-mode scatter kernels (upload), 2 device-tier kernels, 3 D2H memcpy (staged /
   copy mode), 4 H2D memcpy, 5 peer-tier offload kernels, 6 peer-tier upload kernels, 7 direct-mode offload kernels
   (mapped host memory: the whole transfer), 8 direct-mode upload kernels.  bytes = KV payload bytes moved (n * B). */
#define TC_NKINDS 9
typedef struct tc_timing_t {
    double ms[TC_NKINDS];
    int64_t count[TC_NKINDS];
    int64_t bytes[TC_NKINDS];
    /* device-side kernel durations (first CTA start -> last CTA end on %globaltimer, no host launch latency), same
       index; the memcpy kinds (3, 4) stay 0 */
    double kernel_ms[TC_NKINDS];
    int64_t kernel_count[TC_NKINDS];
    int64_t kernel_bytes[TC_NKINDS];
} tc_timing_t;
/* enable: 0 off (the default: zero overhead); 1 event spans around every kernel / memcpy run plus the kernels' own
   start/end timestamps; 2 the kernels' timestamps only (no events: does not perturb the stream schedule); 3 event
   spans around kernel launches only (CUDA events on the launching stream) plus the timestamps.  Other values ->
   TC_E_INVAL.  If out != NULL it receives the totals accumulated since the previous call, which are then
   reset. */
tc_status tc_timing(tc_pool *p, int32_t enable, tc_timing_t *out);
/* Per-span timeline (needs tc_timing enabled): kind as in tc_timing_t, start/end in ms relative to the first span
   after the previous tc_sync, `sync` = index of the sync interval.  out == NULL arms recording of up to `cap`
   records (clearing old ones); otherwise copies up to `cap` records to out, sets *n_out and clears. */
typedef struct tc_span_t {
    int64_t sync;
    int32_t kind;
    double start_ms, end_ms;
    int64_t bytes;
} tc_span_t;
tc_status tc_timeline(tc_pool *p, int64_t cap, tc_span_t *out, int64_t *n_out);
/* Per-call trace (SPEC S:298 trace events offload_done / upload_done with timestamps and block counts):
   one record per offloaded or uploaded handle — op (1 offload, 2 upload), agent, handle, blocks, bytes (n * B), and
   host steady-clock nanoseconds at the call's entry, when its GPU work was enqueued, and when that work completed (a
   cudaLaunchHostFunc callback on the direction's stream; 0 until then; = enqueued on a metadata-only pool).
   tc_trace(p, cap): cap > 0 arms recording of up to cap records (clearing old ones), cap = 0 turns it off.
   tc_trace_read copies up to cap records (call tc_sync first for complete t_done) and clears them. */
typedef struct tc_trace_t {
    int32_t op, agent;
    uint64_t handle;
    int64_t blocks, bytes;
    int64_t t_call_ns, t_enqueued_ns, t_done_ns;
} tc_trace_t;
tc_status tc_trace(tc_pool *p, int64_t cap);
tc_status tc_trace_read(tc_pool *p, tc_trace_t *out, int64_t cap, int64_t *n_out);
const char *tc_strerror(tc_status s);
const char *tc_last_error(tc_pool *p);

/* ---- NEXT-3: Time-Scheduler decision layer (§4.1-4.2), host-only -------------------------------- */
/* FC-duration history of one (agent type, call label): EWMA t_hist after n_obs observations, cold-start estimate
   from static analysis. */
typedef struct tc_fc_stat { double t_hist; int64_t n_obs; double cold_start; } tc_fc_stat;
/* Eq. 1: t_final = alpha*t_req + (1-alpha)*t_hist; t_req < 0 = no developer hint.  Before the first
   observation: the hint if given, else the cold-start estimate. */
double tc_fc_predict(const tc_fc_stat *s, double t_req, double alpha);
/* Feed back an observed duration: first sets t_hist, then t_hist = beta*obs + (1-beta)*t_hist. */
tc_status tc_fc_observe(tc_fc_stat *s, double observed_ms, double beta);
/* T_transfer(n) = T_offload(n) + T_upload(n), linear in the block count. */
typedef struct tc_xfer_model { double offload_ms_per_block, upload_ms_per_block, fixed_ms; } tc_xfer_model;
double tc_transfer_ms(const tc_xfer_model *m, int64_t n_blocks);
/* Calibrate the model from this pool's own measured transfers (needs tc_timing on and at least one tc_sync after
   an offload and an upload; TC_E_BUSY otherwise) — replaces SPEC's paper-derived 60 ms / 4096 blocks.  Per
   direction a least-squares line t = fixed + n * per_block over the link-side spans (through the origin when only
   one size was seen); fixed_ms = the two directions' intercepts. */
tc_status tc_xfer_model_measure(tc_pool *p, tc_xfer_model *m);
typedef struct tc_offload_decision {
    int32_t offload;      /* 1 = offload */
    int32_t match;        /* index of the best-fit waiting request, -1 = none */
    double t_transfer, t_window, n_capacity;
} tc_offload_decision;
/* Alg. 1 ShouldOffload: retain if T_fc <= T_transfer; N_capacity = (T_fc - T_transfer) * v_throughput;
   offload iff some waiting request's token demand fits (best fit = the largest that fits, earliest on ties). */
tc_status tc_should_offload(int64_t n_blocks, double t_fc_ms, double t_transfer_ms, double v_tokens_per_s,
                            const double *waiting_tokens, int64_t n_waiting, tc_offload_decision *out);
typedef struct tc_upload_plan { int32_t immediate; double upload_start, reservation_deadline, predicted_finish; }
    tc_upload_plan;
/* Predictive upload: upload_start = call_start + t_final - upload_ms, gradual reservation ready lead_ms
   before it; if that is before the offload can finish, upload immediately after it. */
tc_status tc_plan_upload(double call_start, double t_final, double upload_ms, double offload_ms, double lead_ms,
                         tc_upload_plan *out);

/* ---- NEXT-3: the Time Scheduler as a runtime (§4.1-4.3; SPEC time_scheduler S:214-304) ------------
   An event machine over a pool, driven by the serving engine with its own clock (ms; reading C2):
     tc_ts_call_start  a function call starts: Eq. 1 forecast over the (agent class, label) EWMA table, T_transfer
                       from params.model, Alg. 1 against the caller's waiting queue; on "offload" the agent's on-GPU
                       blocks are offloaded (tc_offload; NOHOST leaves it retained, reported in out->status) and the
                       predictive upload is planned (tc_plan_upload, lead_ms).
     tc_ts_tick        per agent in id order: begin the gradual reservation reserve_cycles ticks (tick_ms apart)
                       before its deadline (tc_reserve_begin), one tc_reserve_tick, then issue the uploads whose start
                       time has come (tc_upload; NOBLOCKS -> retried at the next tick).
     tc_ts_call_finish the call returned: record the observation (EWMA), then *wait_handle = 0 (retained: resume now)
                       or the upload's handle, uploading immediately if the planned upload was not issued yet (early
                       return).  The engine must tc_wait / tc_stream_wait on that handle before decoding
                       (S:283).  TC_E_NOBLOCKS: no device blocks for the upload yet; nothing else changed; retry.
   Errors: TC_E_INVAL for an unknown agent, a call_start on an agent already in a call, a call_finish on one that is
   not.  Single writer, like the pool. */
typedef struct tc_ts tc_ts;
typedef struct tc_ts_params {
    double alpha, beta;          /* Eq. 1 hint weight, EWMA weight (0.5, 0.5; B10) */
    double cold_start_ms;        /* forecast before any observation and without a hint (100) */
    double lead_ms;              /* reservation ready this long before the upload starts (100) */
    double tick_ms;              /* the engine's scheduling-tick period (10) */
    int32_t reserve_cycles;      /* gradual reservation chunks, 0 = none (4) */
    double v_tokens_per_s;       /* engine throughput for Alg. 1's N_capacity (1000) */
    tc_xfer_model model;         /* T_transfer (default: SPEC's 60 ms round trip per 4096 blocks; better: the
                                    pool's own tc_xfer_model_measure) */
} tc_ts_params;
void tc_ts_params_init(tc_ts_params *prm);
tc_status tc_ts_create(tc_pool *p, const tc_ts_params *prm, tc_ts **out);
void tc_ts_destroy(tc_ts *s);
typedef struct tc_ts_decision {
    int32_t offload;             /* 1 = the agent's blocks were offloaded */
    int32_t match;               /* Alg. 1's best-fit waiting request, -1 = none */
    int32_t status;              /* TC_OK, or TC_E_NOHOST when Alg. 1 said offload but the host buffer refused */
    double t_fc, t_transfer;     /* forecast and T_transfer (ms) */
    double upload_start, reservation_start;   /* plan (engine clock, ms); 0 when retained */
    tc_handle handle;            /* the offload's handle, 0 when retained */
} tc_ts_decision;
tc_status tc_ts_call_start(tc_ts *s, int32_t agent, int32_t label, double now_ms, double t_req_ms,
                           const double *waiting_tokens, int64_t n_waiting, tc_ts_decision *out);
tc_status tc_ts_tick(tc_ts *s, double now_ms, int32_t *uploads_issued);
tc_status tc_ts_call_finish(tc_ts *s, int32_t agent, double now_ms, tc_handle *wait_handle);
/* The forecast table entry of (agent class, label): t_hist and n_obs (0 / 0 before any observation). */
tc_status tc_ts_forecast(tc_ts *s, int32_t agent_class, int32_t label, double *t_hist, int64_t *n_obs);

/* ---- NEXT-4: Space-Scheduler partitions (§5), host-only ------------------------------------------ */
double tc_static_priority(double w_static, int32_t node_depth, int32_t node_out_degree);
/* time_wait * ln(max(tokens_req / max(time_wait, 1 ms), 1)) (clamp: DESIGN.md B7) */
double tc_dynamic_priority(double time_wait_ms, double tokens_req);
/* critical[t] = 1 for the top max(1, floor(ratio * n)) types by score, ties to the lower index (B6). */
tc_status tc_select_critical(int32_t n_types, const double *scores, double critical_ratio, uint8_t *critical);
typedef struct tc_partition_params {
    double gpu_usage_high, gpu_usage_low, adjustment_step, reserve_ratio_max;   /* SPEC: 0.85, 0.50, 0.05, 0.40 */
} tc_partition_params;
/* Alg. 2 UpdateMemoryReservations: Phase 1 adjusts *total_reserve_ratio by usage/tot_blks (clamped to
   [0, reserve_ratio_max]); Phase 2 reserve_num[t] = floor(final_ratio * R_total) for critical types (0 otherwise),
   final_ratio = (usage_t/tot + score_t/S_total)/2, renormalised if they sum above 1 (B8). */
tc_status tc_update_reservations(const tc_partition_params *pp, double *total_reserve_ratio, int64_t usage,
                                 int64_t tot_blks, int32_t n_types, const uint8_t *critical, const double *scores,
                                 const int64_t *type_usage, double *r_total, int64_t *reserve_num);
/* Apply quotas to the pool's classes at once (tc_partition_reserve semantics, all-or-nothing, lazy shrink). */
tc_status tc_apply_reservations(tc_pool *p, int32_t n, const int32_t *classes, const int64_t *reserve_num);

/* ---- NEXT-4 as a runtime: one Space-Scheduler partition update over a pool (SPEC space_scheduler; reading C3) --
   Agent types are the pool's classes.  tc_ss_update: combined score[c] = static_score[c] + sum of
   tc_dynamic_priority over the waiting requests of class c; the top critical_ratio classes are critical
   (tc_select_critical); Alg. 2 (tc_update_reservations) runs on the pool's own usage (non-free blocks; per class the
   on-GPU blocks of its agents) with the persistent total_reserve_ratio; the resulting quotas replace every class's
   reservation at once (non-critical -> 0; lazy shrink).  Outputs (optional, n_classes entries): reserve_num,
   critical flags, combined scores; *total_reserve_ratio = the ratio after Phase 1.  TC_E_INVAL on a waiting class
   out of range.  tc_ss_critical_inversion: 1 iff the evicted class's last combined score is strictly higher than
   the cause's ("critical inversion"). */
typedef struct tc_ss tc_ss;
typedef struct tc_ss_params {
    tc_partition_params partition;   /* 0.85, 0.50, 0.05, 0.40 */
    double critical_ratio;           /* 0.25 */
    double initial_reserve_ratio;    /* 0 */
} tc_ss_params;
void tc_ss_params_init(tc_ss_params *prm);
tc_status tc_ss_create(tc_pool *p, const tc_ss_params *prm, tc_ss **out);
void tc_ss_destroy(tc_ss *s);
tc_status tc_ss_update(tc_ss *s, const double *static_score, int64_t n_waiting, const int32_t *waiting_class,
                       const double *time_wait_ms, const double *tokens_req, int64_t *reserve_num,
                       uint8_t *critical, double *scores, double *total_reserve_ratio);
tc_status tc_ss_critical_inversion(tc_ss *s, int32_t evicted_class, int32_t cause_class, int32_t *inversion);

/* ---- device tier (staged halves; NEXT-2 building block) ---------------------------------------------------- */
/* Gather blocks ids[0..n) into a contiguous device buffer dst[n][L][2][C] (the HBM-bound KG1 kernel), or scatter
   src[n][L][2][C] into blocks ids[0..n) (KS1), on `cuda_stream` (NULL = the offload stream).  No allocator or
   table change: the caller owns the ids' meaning.  dst/src: device (or peer-mapped) pointers, 16-byte aligned. */
tc_status tc_gather_dev(tc_pool *p, const int32_t *ids, int64_t n, void *dst_dev, void *cuda_stream);
tc_status tc_scatter_dev(tc_pool *p, const void *src_dev, const int32_t *ids, int64_t n, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* TOKENCAKE_H */
