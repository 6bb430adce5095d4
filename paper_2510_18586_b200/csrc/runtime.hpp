// Host runtime of the Tokencake offload/upload hot path: block allocator with per-class partitions, CPU block buffer
// (pinned host slots), handles, copy streams + events, descriptor ring and the transfer engine.  Internal C++; the C
// ABI in capi.cpp is the only public surface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tokencake.h"
#include "kernels.cuh"

namespace tc {

enum BlockState : uint8_t { kFree = 0, kAlloc = 1, kPending = 2 };
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

// CPU Block Buffering: one pinned slab cut into fixed block-shard slots + a LIFO free list.
struct HostSlots {
    char *host = nullptr;            // host address of the slab
    char *dev = nullptr;             // device-visible (mapped) address of the same slab
    int64_t count = 0;
    int64_t slot_bytes = 0;
    std::vector<int64_t> free_list;  // back() = next slot handed out
    std::vector<int64_t> released;   // returned to free_list at tc_sync
};

struct AgentRec {
    bool exists = false;
    int32_t cls = 0;
    std::vector<int32_t> table;      // host mirror; -1 = on host
    int32_t live_offloads = 0;       // handles in state OFFLOADED
    int32_t up_event = -1;           // event of the latest upload into this agent since the last sync
};

struct HandleRec {
    int32_t agent = 0, cls = 0;
    std::vector<int32_t> pos;
    std::vector<int64_t> slots;
    int32_t state = kOffloaded;
    int32_t ev = -1;                 // event of its latest transfer, -1 = completed / none
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
    cudaEvent_t ev_compute = nullptr;
    std::vector<cudaStream_t> foreign;       // caller streams used by the device tier
    std::vector<cudaEvent_t> events;         // event pool
    std::vector<int32_t> ev_free, ev_used;

    // pinned descriptor / id ring
    char *ring_host = nullptr, *ring_dev = nullptr;
    int64_t ring_cap = 0, ring_head = 0;

    // transfer modes
    int32_t mode_d2h = TC_XFER_DIRECT, mode_h2d = TC_XFER_DIRECT;
    int ctas_d2h = 0, ctas_h2d = 0, ctas_dev = 0, threads = 256;

    // bookkeeping
    BlockAllocator alloc;
    HostSlots slots;
    std::vector<AgentRec> agents;
    int32_t n_agents = 0;
    std::unordered_map<uint64_t, HandleRec> handles;
    uint64_t next_handle = 1;
    std::vector<std::pair<int32_t, std::vector<int32_t>>> pending_dev;   // (cls, ids) in issue order
    std::vector<uint32_t> stamp;
    uint32_t epoch = 0;

    // optional per-launch timing (tc_timing)
    struct Span {
        int32_t kind;
        cudaEvent_t a, b;
        int64_t bytes;
    };
    bool timing = false;
    std::vector<Span> spans;
    std::vector<cudaEvent_t> tev_free;
    tc_timing_t tacc{};
    cudaEvent_t tev_get();
    tc_status span_begin(cudaStream_t s, cudaEvent_t *a);
    tc_status span_end(cudaStream_t s, int32_t kind, cudaEvent_t a, int64_t bytes);
    void spans_collect();

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
    tc_status query(tc_handle h, bool wait);
    tc_status stream_wait(tc_handle h, cudaStream_t s);
    tc_status sync();
    tc_status fill(uint64_t seed);
    tc_status device_tier(bool gather, const int32_t *ids, int64_t n, void *ext, cudaStream_t s);

    // helpers
    tc_status cuda_fail(cudaError_t e, const char *what);
    int32_t event_get();
    char *ring_alloc(int64_t bytes, char **dev_ptr);
    tc_status enqueue_xfer(bool gather, int32_t mode, const std::vector<XferDesc> &desc,
                           const std::vector<int64_t> &slot_of, cudaStream_t s);
    tc_status table_push(int32_t a, int64_t pos0, int64_t n);
};

}  // namespace tc

struct tc_pool {
    tc::Pool impl;
};
