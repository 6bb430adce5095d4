// Host runtime of the Tokencake offload/upload hot path: block allocator with per-class partitions, CPU block buffer
// (pinned host slots), handles, copy streams + events, the pinned table-push ring and the transfer engine.  Internal C++; the C
// ABI in capi.cpp is the only public surface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tokencake.h"
#include "kernels.cuh"

namespace tc {

enum BlockState : uint8_t { kFree = 0, kAlloc = 1, kPending = 2, kReserved = 3 };
enum HandleState : int32_t { kOffloaded = 1, kUploaded = 2 };

// Lowest-free-id bitmap allocator state + Space-Scheduler partition counters (SURVEY.md §8(c) ops 1-3).
struct BlockAllocator {
    int64_t n = 0;
    std::vector<uint64_t> bits;      // 1 = FREE
    int64_t nfree = 0;
    int64_t hint = 0;                // no FREE bit below word `hint`
    std::vector<uint8_t> state;
    std::vector<int32_t> own_agent, own_pos;
    std::vector<int64_t> reserved, claimed;

    void init(int64_t n_blocks, int n_classes);
    int64_t unclaimed(int c) const { return reserved[c] > claimed[c] ? reserved[c] - claimed[c] : 0; }
    int64_t unclaimed_sum() const;
    // Partition rule on explicit counters (used for dry runs): returns r (blocks from the reservation) or -1.
    static int64_t plan(int c, int64_t n, int64_t nfree, const std::vector<int64_t> &reserved,
                        const std::vector<int64_t> &claimed);
    void take_lowest(int64_t k, int32_t *out);   // clears the k lowest FREE bits, ascending
    void set_free(int32_t b);
};

// CPU Block Buffering: one pinned slab cut into fixed block-shard slots + their free set.  Build choice
// (reading A16'): a batch's slots are one contiguous run of the slab whenever one is free (lowest address
// first), so the batch crosses the host link as one DMA per staging piece; otherwise the lowest free slots.  Slot
// identity is outside the parity contract (A4); only counts are compared with the oracle's LIFO list.
struct HostSlots {
    char *host = nullptr;            // host address of the slab
    char *dev = nullptr;             // device-visible (mapped) address of the same slab
    int64_t count = 0;
    int64_t slot_bytes = 0;
    std::vector<uint64_t> bits;      // 1 = free
    int64_t nfree = 0;
    std::vector<int64_t> released;   // returned to the free set at a retirement point (tc_sync / tc_retire)
    std::vector<uint32_t> released_epoch;   // retirement epoch each released slot was created in

    void init(int64_t S);
    // n free slots: the lowest contiguous run of n if one exists, else the n lowest free slots.  No state change.
    void choose(int64_t n, int64_t *out) const;
    void take(const int64_t *s, int64_t n);
    void give(int64_t s) {
        bits[s >> 6] |= 1ull << (s & 63);
        ++nfree;
    }
};

// NEXT-2 peer tier: block-shard slots in a neighbouring GPU's HBM, ids S .. S+count-1, own LIFO free list.
struct PeerSlots {
    char *dev = nullptr;             // base of the slab on `device` (peer-accessible from the pool's device)
    int device = -1;
    int64_t count = 0;
    std::vector<int64_t> free_list;  // back() = next slot handed out
};

struct AgentRec {
    bool exists = false;
    int32_t cls = 0;
    std::vector<int32_t> table;      // host mirror; -1 = on host
    int32_t live_offloads = 0;       // handles in state OFFLOADED
    int32_t up_event = -1;           // event of the latest upload into this agent since the last sync
    cudaEvent_t push_ev = nullptr;   // latest block-table push for this agent on s_off (no compute stream set)
};

struct HandleRec {
    int32_t agent = 0, cls = 0;
    std::vector<int32_t> pos;
    std::vector<int64_t> slots;
    int32_t state = kOffloaded;
    int32_t ev = -1;                 // event of its latest transfer, -1 = completed / none
    std::vector<int64_t> plan;       // gradual reservation: chunk per tick (empty = none active)
    int32_t ticks = 0;
    std::vector<int32_t> resv;       // destination blocks claimed so far, in claim order
    uint32_t up_epoch = 0;           // retirement epoch of its upload (forgotten once that epoch retires)
};

struct Pool {
    // geometry
    int32_t L = 0, H = 0, Hl = 0, D = 0, T = 0, rank = 0, world = 1;
    tc_dtype dtype = TC_BF16;
    int64_t N = 0, C = 0, B = 0;
    int32_t n_classes = 8, max_agents = 1024, max_bpa = 4096;
    bool meta_only = false;
    int device = -1;

    // device memory
    char *kv = nullptr;
    bool kv_owned = false;
    int32_t *table_dev = nullptr;
    bool table_owned = false;
    char *staging[2] = {nullptr, nullptr};   // [0] = D2H, [1] = H2D
    int64_t staging_bytes = 0;

    // streams / events
    cudaStream_t s_up = nullptr, s_off = nullptr, s_compute = nullptr;
    cudaStream_t s_up_k = nullptr, s_off_k = nullptr;   // staged mode: device-side kernels of each direction
    // cross-batch double buffering of the staging buffer (single-piece batches that fit half of it): batch k of a
    // direction uses half k % 2, so its kernel / DMA need not wait for batch k-1's DMA / kernel on the other half
    bool halves = true;
    int32_t half_next[2] = {0, 0};                      // per direction: the half the next batch uses
    cudaEvent_t half_free[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [dir][half]: last use done
    int64_t piece_bytes = 256ll << 20;                  // staged pipeline: large pieces
    int64_t head_bytes = 0;                             // > 0: a small first (offload) / last (upload) piece
    cudaEvent_t ev_compute = nullptr;
    // caller streams the device tier ran on: an event recorded behind each such launch (the pool never holds the
    // caller's stream handle, which the caller may destroy); tc_sync / tc_timing / ring wraps wait on these events
    std::vector<cudaEvent_t> fev_live, fev_free;
    tc_status drain_foreign();
    std::vector<cudaEvent_t> events;         // event pool
    std::vector<int32_t> ev_free, ev_used;

    // pinned mapped ring for host->device block-table pushes (decode growth); kernel descriptors travel by value
    char *ring_host = nullptr, *ring_dev = nullptr;
    int64_t ring_cap = 0, ring_head = 0;

    // transfer modes
    int32_t mode_d2h = TC_XFER_DIRECT, mode_h2d = TC_XFER_DIRECT;
    bool auto_dir[2] = {false, false};        // the direction's mode came from AUTO (small batches go DIRECT)
    int32_t auto_choice[2] = {TC_XFER_STAGED, TC_XFER_STAGED};   // what AUTO resolves to (tc_calibrate)
    tc_status calibrate(int64_t probe_bytes, tc_calibration_t *out);
    tc_status calibrate_small(int64_t k, const std::vector<XferDesc> &da, const std::vector<XferDesc> &db,
                              const std::vector<int64_t> &sa, const std::vector<int64_t> &sb, tc_calibration_t *out);
    int64_t auto_direct_bytes[2] = {2ll << 20, 2ll << 20};   // per direction: AUTO batches up to this go DIRECT
    // launch config per path: [0] direct D2H, [1] direct H2D, [2] device tier + staged kernels, [3] peer tier
    int ctas[4] = {0, 0, 0, 0}, nthreads[4] = {256, 256, 256, 256}, variant[4] = {0, 0, 3, 3};

    // bookkeeping
    BlockAllocator alloc;
    HostSlots slots;
    PeerSlots peer;
    bool is_peer(int64_t slot) const { return peer.count > 0 && slot >= slots.count; }
    char *peer_ptr(int64_t slot) const { return peer.dev + (slot - slots.count) * B; }
    std::vector<AgentRec> agents;
    int32_t n_agents = 0;
    std::unordered_map<uint64_t, HandleRec> handles;
    uint64_t next_handle = 1;
    std::vector<std::pair<int32_t, std::vector<int32_t>>> pending_dev;   // (cls, ids) in issue order
    std::vector<uint32_t> pending_epoch;     // retirement epoch of each pending entry (reading A8')
    uint32_t epoch_id = 0;                   // retirement points (tc_sync / tc_retire) so far
    std::vector<uint32_t> ev_epoch;          // per event index: the epoch it was last handed out in
    tc_status retire(int32_t lag = 1);       // tc_retire(_lag): retire what was enqueued before the lag-th previous point
    void retire_before(uint32_t upto);
    std::vector<uint32_t> stamp;
    uint32_t epoch = 0;

    // optional per-launch timing (tc_timing)
    struct Span {
        int32_t kind;
        cudaEvent_t a, b;
        int64_t bytes;
        bool link;                           // host-link side of a transfer (DMA or direct kernel)
    };
    int32_t timing = 0;   // 0 off, 1 event spans + kernel timestamps, 2 kernel timestamps, 3 kernel spans + timestamps
    std::vector<Span> spans;
    std::vector<cudaEvent_t> tev_free;
    tc_timing_t tacc{};
    cudaEvent_t tev_get();
    tc_status span_begin(cudaStream_t s, cudaEvent_t *a, bool kernel = true);
    bool span_on(bool kernel) const;
    tc_status span_end(cudaStream_t s, int32_t kind, cudaEvent_t a, int64_t bytes, bool link = true);
    void spans_collect();
    bool check = false;                      // TC_CHECK=1: invariants after every mutating call
    void check_invariants(const char *after) const;
    // TC_CHECK: every descriptor of a launch addresses a pool block, a table entry and a whole block image inside the
    // buffer its kind writes to / reads from (staging, host slab, peer slab); aborts on a violation
    void check_descs(int32_t kind, const XferDesc *d, int64_t n) const;
    void stamps_collect();
    std::vector<tc_span_t> timeline;         // per-span records (tc_timeline), capped
    // per-call trace (tc_trace): records live in a fixed array so the completion callbacks can fill t_done in place
    std::unique_ptr<tc_trace_t[]> trace_buf;
    int64_t trace_cap = 0, trace_n = 0;
    int64_t trace_t0 = 0;                    // t_call of the call being enqueued
    void trace_calls(int32_t op, const int32_t *agents, const tc_handle *hs, const int64_t *off, int32_t k,
                     cudaStream_t s);
    int64_t timeline_cap = 0;
    int64_t sync_count = 0;
    static constexpr int64_t kKts = 65536;   // kernel stamp slots between collections
    unsigned long long *kts_dev = nullptr;   // device {start, end} %globaltimer pairs, one per timed launch
    std::vector<unsigned long long> kts_init;
    std::vector<std::pair<int32_t, int64_t>> kts_meta;   // (kind, bytes) per used pair
    bool kts_ensure();
    XferGeom geom(int32_t kind, int64_t bytes);
    // link-side transfer spans per direction, for the least-squares fit t = fixed + n * per_block
    // (tc_xfer_model_measure): sums of 1, n, t, n*n, n*t over the spans
    double cal_ms[2] = {0, 0};
    int64_t cal_blocks[2] = {0, 0};
    double cal_cnt[2] = {0, 0}, cal_nn[2] = {0, 0}, cal_nt[2] = {0, 0};

    // counters / errors
    int64_t n_launch = 0, n_memcpy = 0, bytes_d2h = 0, bytes_h2d = 0;
    bool cuda_dead = false;
    std::string last_error;

    ~Pool();
    tc_status create(const tc_pool_desc &d);

    tc_status reserve(int32_t c, int64_t n);
    tc_status agent_add(int32_t a, int32_t c);
    tc_status alloc_blocks(int32_t a, int64_t n, int32_t *out);
    tc_status agent_free(int32_t a);
    tc_status offload_batch(int32_t na, const int32_t *agents, const int64_t *offsets, const int32_t *ids,
                            tc_handle *out);
    tc_status upload_batch(int32_t nh, const tc_handle *hs, const int64_t *offsets, int32_t *out_ids);
    tc_status cycle(int32_t nh, const tc_handle *hs, const int64_t *up_off, int32_t *out_ids, int32_t na,
                    const int32_t *ags, const int64_t *off_off, const int32_t *ids, tc_handle *out_h);
    // A batch's blocks split by tier: host-tier descriptors + slots (copy engine / direct kernel) and peer-tier
    // descriptors (ext = the peer slot's device address; one device-side kernel).
    struct TierSplit {
        std::vector<XferDesc> hdesc, pdesc;
        std::vector<int64_t> hslot;
    };
    struct OffPlan {
        int32_t na = 0;
        const int32_t *ags = nullptr, *ids = nullptr;
        const int64_t *off = nullptr;
        std::vector<XferDesc> desc;
        std::vector<int64_t> slot_of;
        int64_t host_taken = 0, peer_taken = 0;
        std::vector<int64_t> host_slots;     // the batch's host-tier slots, in item order (HostSlots::choose)
        TierSplit ts;
        // commit-time records built at plan time, so commit_offload allocates nothing (strong guarantee on OOM)
        std::unordered_map<tc_handle, HandleRec> newh;
        std::vector<std::vector<int32_t>> pend;
    };
    struct UpPlan {
        int32_t nh = 0;
        const tc_handle *hs = nullptr;
        const int64_t *off = nullptr;
        std::vector<HandleRec *> hr;
        std::vector<int64_t> rr, need;
        int64_t n_fresh = 0;
        std::vector<int32_t> dst;
        std::vector<XferDesc> desc;
        std::vector<int64_t> slot_of;
        TierSplit ts;
        std::vector<int32_t> taken;          // scratch for commit_upload's take_lowest (allocated at plan time)
    };
    void split_tiers(const std::vector<XferDesc> &desc, const std::vector<int64_t> &slot_of, TierSplit &ts) const;
    tc_status peer_launch(bool gather, const std::vector<XferDesc> &pd, cudaStream_t s, int32_t *join_ev);
    tc_status join(cudaStream_t s, int32_t ev);
    tc_status plan_offload(OffPlan &P, int32_t na, const int32_t *ags, const int64_t *off, const int32_t *ids);
    // GPU-side dependencies of an offload; ups = also the agents' last uploads (false: the job waits per piece)
    tc_status offload_waits(const OffPlan &P, bool ups = true);
    // ev = the batch's completion event; item_ev (optional) = per-item completion events (fine-grained jobs)
    void commit_offload(OffPlan &P, int32_t ev, tc_handle *out, const std::vector<int32_t> *item_ev = nullptr);
    tc_status plan_upload(UpPlan &P, int32_t nh, const tc_handle *hs, const int64_t *off);
    tc_status upload_waits(const UpPlan &P);
    void commit_upload(UpPlan &P, int32_t ev, int32_t *out_ids, const std::vector<int32_t> *item_ev = nullptr);
    tc_status query(tc_handle h, bool wait);
    tc_status stream_wait(tc_handle h, cudaStream_t s);
    tc_status sync();
    tc_status fill(uint64_t seed);
    tc_status reserve_begin(tc_handle h, int32_t cycles);
    tc_status reserve_tick();
    tc_status reserve_cancel(tc_handle h);
    std::set<tc_handle> resv_active;         // handles with an active gradual reservation, issue order
    int64_t n_reserved = 0;
    tc_status device_tier(bool gather, const int32_t *ids, int64_t n, void *ext, cudaStream_t s);

    // helpers
    tc_status cuda_fail(cudaError_t e, const char *what);
    tc_status enqueue_oom();
    int32_t event_get();
    char *ring_alloc(int64_t bytes, char **dev_ptr);
    tc_status enqueue_xfer(bool gather, int32_t mode, const std::vector<XferDesc> &desc,
                           const std::vector<int64_t> &slot_of, cudaStream_t s);
    // two-phase transfer job (see runtime.cpp)
    struct XferJob {
        bool gather = false, ring_reuse = false;
        int32_t half = -1;                   // >= 0: cross-batch double buffering on this staging half
        int32_t mode = TC_XFER_DIRECT;
        const std::vector<XferDesc> *desc = nullptr;
        const std::vector<int64_t> *slot_of = nullptr;
        cudaStream_t s = nullptr, sk = nullptr;
        int64_t n = 0, npieces = 0;
        std::vector<int64_t> cut;            // piece p = blocks [cut[p], cut[p+1])
        char *stg = nullptr;
        std::vector<int32_t> ev;
        bool need_hop = false;               // the aux stream starts after the main stream's waits (phase A)
        int64_t pb = 0;                      // ring reuse: blocks per staging half (pieces are at most this)
        // Fine-grained dependencies (a staged batch of several pieces): item k (one agent's offload / one handle's
        // upload) = blocks [item_off[k], item_off[k+1]); a piece waits only for item_dep[] of the items it holds,
        // and piece_done[p] marks the end of piece p's whole transfer (the items' completion events).
        const int64_t *item_off = nullptr;
        const int32_t *item_dep = nullptr;
        int32_t n_items = 0;
        std::vector<int32_t> piece_done;
    };
    bool fine_off = false;                   // TC_FINE_DEPS=0: batch-granular dependencies (A/B)
    tc_status piece_waits(const XferJob &j, int64_t a, int64_t b, cudaStream_t st);
    // fine-grained mode for a job after xfer_init (staged, several pieces, no peer-tier part); deps per item
    bool fine_grained(XferJob &j, const int64_t *item_off, int32_t n_items, const std::vector<int32_t> &deps);
    void item_events(const XferJob &j, std::vector<int32_t> &out) const;
    char *xfer_base(const XferJob &j, int64_t p) const;
    // host address (and its device mapping) of a host slot id: the CPU block buffer, or an ablation slab
    char *host_ptr(int64_t slot) const;
    char *host_dev_ptr(int64_t slot) const;
    // Fig. 11 ablation (tc_pool_desc.unbuffered): per-offload pinned slabs instead of the CPU block buffer
    struct ExtraSlab {
        char *host, *dev;
        int64_t n, live;
    };
    bool unbuffered = false;
    std::map<int64_t, ExtraSlab> extra;      // first slot id -> slab
    int64_t next_slot = 0;
    // item_off (optional, n_items + 1 block offsets): piece cuts fall on item boundaries where they can (below)
    tc_status xfer_init(XferJob &j, bool gather, int32_t mode, const std::vector<XferDesc> *desc,
                        const std::vector<int64_t> *slot_of, cudaStream_t s, const int64_t *item_off = nullptr,
                        int32_t n_items = 0);
    int64_t min_piece_bytes = 64ll << 20;    // an item-aligned cut never leaves a piece smaller than this
    tc_status xfer_phase_a(XferJob &j);
    tc_status xfer_phase_b(XferJob &j);
    tc_status xfer_copy(XferJob &j, int64_t a, int64_t b, char *base);
    tc_status xfer_kernel(XferJob &j, int64_t a, int64_t b, char *base);
    tc_status xfer_copy2d(XferJob &j);
    int32_t auto_mode(int dir) const;
    tc_status launch_descs(bool gather, int32_t kind, int path, const XferDesc *d, int64_t n, cudaStream_t s);
    std::vector<XferDesc> cd_;               // scratch: descriptors of the launch being built
    tc_status ev_rec(cudaStream_t st, int32_t *out);
    std::vector<void *> cp_dst, cp_src;
    std::vector<size_t> cp_size;
    tc_status table_push(int32_t a, int64_t pos0, int64_t n);
};

}  // namespace tc

struct tc_pool {
    tc::Pool impl;
};
