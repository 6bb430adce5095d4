// C ABI of the Tokencake offload/upload hot path (include/tokencake.h): argument marshalling, status mapping and
// exception containment around the runtime in runtime.cpp.  No C++ exception crosses this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include <nvtx3/nvToolsExt.h>

#include "runtime.hpp"

using tc::Pool;

// Mutating entry points: an NVTX range named after the call (visible in Nsight Systems / ncu), and with TC_CHECK=1
// the SPEC invariants re-checked after the call (Pool::check_invariants).
namespace {
struct Mut {
    const Pool &p;
    const char *name;
    Mut(const Pool &p_, const char *n) : p(p_), name(n) { nvtxRangePushA(n); }
    ~Mut() {
        nvtxRangePop();
        if (p.check) p.check_invariants(name);
    }
};
}  // namespace
#define TC_MUT(name) Mut mut_(P, name)

#define TC_GUARD(p)                         \
    if (!(p)) return TC_E_INVAL;            \
    Pool &P = (p)->impl;                    \
    (void)P;                                \
    try
#define TC_CATCH                                              \
    catch (const std::bad_alloc &) { return TC_E_OOM; }       \
    catch (...) { return TC_E_INVAL; }

extern "C" {

void tc_pool_desc_init(tc_pool_desc *d, int32_t layers, int32_t kv_heads, int32_t head_dim, int32_t block_tokens,
                       tc_dtype dtype, int64_t n_blocks) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->layers = layers;
    d->kv_heads = kv_heads;
    d->head_dim = head_dim;
    d->block_tokens = block_tokens;
    d->dtype = dtype;
    d->n_blocks = n_blocks;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    d->device = dev;
    d->shard_rank = 0;
    d->shard_world = 1;
    d->xfer_d2h = TC_XFER_AUTO;
    d->xfer_h2d = TC_XFER_AUTO;
    d->peer_device = -1;
    d->peer_slots = 0;
}

tc_status tc_pool_create_ex(const tc_pool_desc *d, tc_pool **out) {
    if (!d || !out) return TC_E_INVAL;
    tc_pool *p = nullptr;
    try {
        p = new tc_pool();
        const tc_status st = p->impl.create(*d);
        if (st != TC_OK) {
            delete p;
            return st;
        }
    } catch (const std::bad_alloc &) {
        delete p;
        return TC_E_OOM;
    }
    *out = p;
    return TC_OK;
}

tc_status tc_pool_create(int32_t layers, int32_t kv_heads, int32_t head_dim, int32_t block_tokens, tc_dtype dtype,
                         int64_t n_blocks, tc_pool **out) {
    tc_pool_desc d;
    tc_pool_desc_init(&d, layers, kv_heads, head_dim, block_tokens, dtype, n_blocks);
    return tc_pool_create_ex(&d, out);
}

void tc_pool_destroy(tc_pool *p) { delete p; }

tc_status tc_pool_kv(tc_pool *p, void **kv_dev, int64_t *chunk_bytes) {
    TC_GUARD(p) {
        if (P.meta_only) return TC_E_NODEV;
        if (kv_dev) *kv_dev = P.kv;
        if (chunk_bytes) *chunk_bytes = P.C;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_set_compute_stream(tc_pool *p, void *cuda_stream) {
    TC_GUARD(p) {
        P.s_compute = static_cast<cudaStream_t>(cuda_stream);
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_streams(tc_pool *p, void **upload_stream, void **offload_stream) {
    TC_GUARD(p) {
        if (P.meta_only) return TC_E_NODEV;
        if (upload_stream) *upload_stream = P.s_up;
        if (offload_stream) *offload_stream = P.s_off;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_set_xfer_mode(tc_pool *p, int32_t d2h, int32_t h2d) {
    TC_GUARD(p) {
        if (d2h < 0 || d2h > 3 || h2d < 0 || h2d > 3) return TC_E_INVAL;
        P.auto_dir[0] = d2h == TC_XFER_AUTO;
        P.auto_dir[1] = h2d == TC_XFER_AUTO;
        P.mode_d2h = P.auto_dir[0] ? P.auto_mode(0) : d2h;
        P.mode_h2d = P.auto_dir[1] ? P.auto_mode(1) : h2d;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_calibrate(tc_pool *p, int64_t probe_bytes, tc_calibration_t *out) {
    TC_GUARD(p) {
        TC_MUT("tc_calibrate");
        return P.calibrate(probe_bytes, out);
    }
    TC_CATCH
}

tc_status tc_set_launch_config(tc_pool *p, int32_t path, int32_t ctas, int32_t threads, int32_t variant) {
    TC_GUARD(p) {
        if (path < 0 || path > 3 || threads < 32 || threads > 256 || threads % 32 || variant < 0 || variant > 4)
            return TC_E_INVAL;
        P.ctas[path] = ctas;
        P.nthreads[path] = threads;
        P.variant[path] = variant;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_fill_kv(tc_pool *p, uint64_t seed) {
    TC_GUARD(p) { return P.fill(seed); }
    TC_CATCH
}

tc_status tc_partition_reserve(tc_pool *p, int32_t agent_class, int64_t n_blocks) {
    TC_GUARD(p) {
        TC_MUT("tc_partition_reserve");
        return P.reserve(agent_class, n_blocks);
    }
    TC_CATCH
}

tc_status tc_agent_add(tc_pool *p, int32_t agent, int32_t agent_class) {
    TC_GUARD(p) {
        TC_MUT("tc_agent_add");
        return P.agent_add(agent, agent_class);
    }
    TC_CATCH
}

tc_status tc_alloc(tc_pool *p, int32_t agent, int64_t n, int32_t *out_ids) {
    TC_GUARD(p) {
        if (!out_ids) return TC_E_INVAL;
        TC_MUT("tc_alloc");
        return P.alloc_blocks(agent, n, out_ids);
    }
    TC_CATCH
}

tc_status tc_agent_free(tc_pool *p, int32_t agent) {
    TC_GUARD(p) {
        TC_MUT("tc_agent_free");
        return P.agent_free(agent);
    }
    TC_CATCH
}

tc_status tc_offload(tc_pool *p, int32_t agent, const int32_t *block_ids, int64_t n, tc_handle *out) {
    const int64_t off[2] = {0, n};
    TC_GUARD(p) {
        TC_MUT("tc_offload");
        return P.offload_batch(1, &agent, off, block_ids, out);
    }
    TC_CATCH
}

tc_status tc_upload(tc_pool *p, tc_handle h, int32_t *out_new_ids) {
    TC_GUARD(p) {
        auto it = P.handles.find(h);
        if (it == P.handles.end() || it->second.state != tc::kOffloaded) return TC_E_HANDLE;
        const int64_t off[2] = {0, (int64_t)it->second.pos.size()};
        TC_MUT("tc_upload");
        return P.upload_batch(1, &h, off, out_new_ids);
    }
    TC_CATCH
}

tc_status tc_offload_batch(tc_pool *p, int32_t n_agents, const int32_t *agents, const int64_t *offsets,
                           const int32_t *block_ids, tc_handle *out_handles) {
    TC_GUARD(p) {
        TC_MUT("tc_offload_batch");
        return P.offload_batch(n_agents, agents, offsets, block_ids, out_handles);
    }
    TC_CATCH
}

tc_status tc_upload_batch(tc_pool *p, int32_t n_handles, const tc_handle *hs, const int64_t *offsets,
                          int32_t *out_new_ids) {
    TC_GUARD(p) {
        TC_MUT("tc_upload_batch");
        return P.upload_batch(n_handles, hs, offsets, out_new_ids);
    }
    TC_CATCH
}

tc_status tc_cycle(tc_pool *p, int32_t n_handles, const tc_handle *hs, const int64_t *up_offsets,
                   int32_t *out_new_ids, int32_t n_agents, const int32_t *agents, const int64_t *off_offsets,
                   const int32_t *block_ids, tc_handle *out_handles) {
    TC_GUARD(p) {
        TC_MUT("tc_cycle");
        return P.cycle(n_handles, hs, up_offsets, out_new_ids, n_agents, agents, off_offsets, block_ids,
                       out_handles);
    }
    TC_CATCH
}

tc_status tc_reserve_begin(tc_pool *p, tc_handle h, int32_t cycles) {
    TC_GUARD(p) {
        TC_MUT("tc_reserve_begin");
        return P.reserve_begin(h, cycles);
    }
    TC_CATCH
}

tc_status tc_reserve_tick(tc_pool *p) {
    TC_GUARD(p) {
        TC_MUT("tc_reserve_tick");
        return P.reserve_tick();
    }
    TC_CATCH
}

tc_status tc_reserve_cancel(tc_pool *p, tc_handle h) {
    TC_GUARD(p) {
        TC_MUT("tc_reserve_cancel");
        return P.reserve_cancel(h);
    }
    TC_CATCH
}

tc_status tc_reserve_info(tc_pool *p, tc_handle h, int64_t *reserved, int64_t *total) {
    TC_GUARD(p) {
        auto it = P.handles.find(h);
        if (it == P.handles.end()) return TC_E_HANDLE;
        if (reserved) *reserved = (int64_t)it->second.resv.size();
        if (total) *total = (int64_t)it->second.pos.size();
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_query(tc_pool *p, tc_handle h) {
    TC_GUARD(p) { return P.query(h, false); }
    TC_CATCH
}

tc_status tc_wait(tc_pool *p, tc_handle h) {
    TC_GUARD(p) { return P.query(h, true); }
    TC_CATCH
}

tc_status tc_stream_wait(tc_pool *p, tc_handle h, void *cuda_stream) {
    TC_GUARD(p) { return P.stream_wait(h, static_cast<cudaStream_t>(cuda_stream)); }
    TC_CATCH
}

tc_status tc_retire(tc_pool *p) {
    TC_GUARD(p) {
        TC_MUT("tc_retire");
        return P.retire();
    }
    TC_CATCH
}

tc_status tc_retire_lag(tc_pool *p, int32_t lag) {
    TC_GUARD(p) {
        TC_MUT("tc_retire_lag");
        return P.retire(lag);
    }
    TC_CATCH
}

tc_status tc_sync(tc_pool *p) {
    TC_GUARD(p) {
        TC_MUT("tc_sync");
        return P.sync();
    }
    TC_CATCH
}

tc_status tc_block_table(tc_pool *p, int32_t agent, int32_t *out, int64_t cap, int64_t *n_out) {
    TC_GUARD(p) {
        if (agent < 0 || agent >= P.max_agents || !P.agents[agent].exists || !n_out) return TC_E_INVAL;
        const auto &t = P.agents[agent].table;
        *n_out = (int64_t)t.size();
        if (out) {
            if (cap < (int64_t)t.size()) return TC_E_INVAL;
            std::memcpy(out, t.data(), t.size() * sizeof(int32_t));
        }
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_block_table_dev(tc_pool *p, int32_t **dev_table, int64_t *row_stride) {
    TC_GUARD(p) {
        if (P.meta_only) return TC_E_NODEV;
        if (dev_table) *dev_table = P.table_dev;
        if (row_stride) *row_stride = P.max_bpa;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_handle_info(tc_pool *p, tc_handle h, int32_t *agent, int64_t *n, int32_t *state) {
    TC_GUARD(p) {
        auto it = P.handles.find(h);
        if (it == P.handles.end()) return TC_E_HANDLE;
        if (agent) *agent = it->second.agent;
        if (n) *n = (int64_t)it->second.pos.size();
        if (state) *state = it->second.state;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_handle_host(tc_pool *p, tc_handle h, int64_t i, const void **host_ptr) {
    TC_GUARD(p) {
        if (P.meta_only) return TC_E_NODEV;
        auto it = P.handles.find(h);
        if (it == P.handles.end() || it->second.state != tc::kOffloaded) return TC_E_HANDLE;
        if (i < 0 || i >= (int64_t)it->second.slots.size() || !host_ptr) return TC_E_INVAL;
        if (P.is_peer(it->second.slots[i])) return TC_E_INVAL;   // a peer-tier slot has no host address
        *host_ptr = P.host_ptr(it->second.slots[i]);
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_handle_read(tc_pool *p, tc_handle h, int64_t i, void *dst, int32_t *tier) {
    TC_GUARD(p) {
        if (P.meta_only) return TC_E_NODEV;
        auto it = P.handles.find(h);
        if (it == P.handles.end() || it->second.state != tc::kOffloaded) return TC_E_HANDLE;
        if (i < 0 || i >= (int64_t)it->second.slots.size() || !dst) return TC_E_INVAL;
        const tc_status st = P.query(h, /*wait=*/true);
        if (st != TC_OK) return st;
        const int64_t slot = it->second.slots[i];
        const bool pe = P.is_peer(slot);
        if (tier) *tier = pe ? 1 : 0;
        if (!pe) {
            std::memcpy(dst, P.host_ptr(slot), (size_t)P.B);
            return TC_OK;
        }
        if (cudaMemcpy(dst, P.peer_ptr(slot), (size_t)P.B, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return TC_E_CUDA;
        }
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_stats(tc_pool *p, tc_stats_t *s) {
    TC_GUARD(p) {
        if (!s) return TC_E_INVAL;
        std::memset(s, 0, sizeof(*s));
        s->n_blocks = P.N;
        s->free_blocks = P.alloc.nfree;
        int64_t pend = 0;
        for (auto &pc : P.pending_dev) pend += (int64_t)pc.second.size();
        s->pending_blocks = pend;
        s->alloc_blocks = P.N - P.alloc.nfree - pend - P.n_reserved;
        s->reserved_blocks = P.n_reserved;
        s->host_slots = P.slots.count;
        s->host_free = P.slots.nfree;
        s->host_released = (int64_t)P.slots.released.size();
        s->host_used = P.slots.count - s->host_free - s->host_released;
        s->chunk_bytes = P.C;
        s->block_bytes = P.B;
        s->n_classes = P.n_classes;
        s->n_agents = P.n_agents;
        for (int c = 0; c < P.n_classes; ++c) {
            s->reserved[c] = P.alloc.reserved[c];
            s->claimed[c] = P.alloc.claimed[c];
        }
        int64_t live = 0;
        for (auto &kv : P.handles) live += kv.second.state == tc::kOffloaded;
        s->live_handles = live;
        s->kernel_launches = P.n_launch;
        s->memcpy_calls = P.n_memcpy;
        s->bytes_d2h = P.bytes_d2h;
        s->bytes_h2d = P.bytes_h2d;
        s->xfer_d2h = P.mode_d2h;
        s->xfer_h2d = P.mode_h2d;
        s->peer_slots = P.peer.count;
        s->peer_free = (int64_t)P.peer.free_list.size();
        int64_t prel = 0, hrel = 0;
        for (int64_t x : P.slots.released) (P.is_peer(x) ? prel : hrel) += 1;
        s->peer_used = P.peer.count - s->peer_free - prel;
        s->host_used = P.slots.count - s->host_free - hrel;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_timing(tc_pool *p, int32_t enable, tc_timing_t *out) {
    TC_GUARD(p) {
        if (enable < 0 || enable > 3) return TC_E_INVAL;
        if (!P.meta_only && (!P.kts_meta.empty() || !P.spans.empty())) {   // collected lazily (runtime.cpp)
            for (cudaStream_t s : {P.s_up, P.s_off, P.s_up_k, P.s_off_k})
                if (cudaStreamSynchronize(s) != cudaSuccess) return P.cuda_fail(cudaGetLastError(), "timing sync");
            if (tc_status st = P.drain_foreign(); st != TC_OK) return st;
            P.spans_collect();
            P.stamps_collect();
        }
        P.timing = P.meta_only ? 0 : enable;
        if (P.timing) P.kts_ensure();                   // allocate now, not at the first timed launch
        if (P.timing == 1 || P.timing == 3) {           // span events created now, not inside a timed loop
            while (P.tev_free.size() < 1024) {
                cudaEvent_t e = nullptr;
                if (cudaEventCreate(&e) != cudaSuccess) return P.cuda_fail(cudaGetLastError(), "timing events");
                P.tev_free.push_back(e);
            }
            P.spans.reserve(512);
        }
        if (out) {
            *out = P.tacc;
            P.tacc = tc_timing_t{};
        }
        return TC_OK;
    }
    TC_CATCH
}

// Drain every stream the pool uses (trace records are written by host callbacks queued on them).
static tc_status drain(Pool &P) {
    if (P.meta_only) return TC_OK;
    for (cudaStream_t s : {P.s_up, P.s_off, P.s_up_k, P.s_off_k})
        if (cudaStreamSynchronize(s) != cudaSuccess) return P.cuda_fail(cudaGetLastError(), "drain");
    return TC_OK;
}

tc_status tc_trace(tc_pool *p, int64_t cap) {
    TC_GUARD(p) {
        if (cap < 0) return TC_E_INVAL;
        const tc_status st = drain(P);
        if (st != TC_OK) return st;
        P.trace_buf.reset(cap > 0 ? new tc_trace_t[cap] : nullptr);
        P.trace_cap = cap;
        P.trace_n = 0;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_trace_read(tc_pool *p, tc_trace_t *out, int64_t cap, int64_t *n_out) {
    TC_GUARD(p) {
        if (!out || !n_out || cap < 0) return TC_E_INVAL;
        const tc_status st = drain(P);
        if (st != TC_OK) return st;
        const int64_t n = std::min(cap, P.trace_n);
        if (n > 0) std::memcpy(out, P.trace_buf.get(), (size_t)n * sizeof(tc_trace_t));
        *n_out = n;
        P.trace_n = 0;
        return TC_OK;
    }
    TC_CATCH
}

tc_status tc_timeline(tc_pool *p, int64_t cap, tc_span_t *out, int64_t *n_out) {
    TC_GUARD(p) {
        if (!n_out) return TC_E_INVAL;
        if (!out) {                                  // (re)arm: keep up to `cap` records from now on
            P.timeline.clear();
            P.timeline_cap = cap;
            *n_out = 0;
            return TC_OK;
        }
        const int64_t n = std::min<int64_t>(cap, (int64_t)P.timeline.size());
        std::memcpy(out, P.timeline.data(), (size_t)n * sizeof(tc_span_t));
        *n_out = n;
        P.timeline.clear();
        return TC_OK;
    }
    TC_CATCH
}

const char *tc_strerror(tc_status s) {
    switch (s) {
        case TC_OK: return "ok";
        case TC_E_INVAL: return "invalid argument";
        case TC_E_NOBLOCKS: return "not enough free device blocks under the partition rule";
        case TC_E_NOHOST: return "host block buffer exhausted";
        case TC_E_HANDLE: return "unknown or already-uploaded handle";
        case TC_E_BUSY: return "busy";
        case TC_E_CUDA: return "CUDA error";
        case TC_E_OOM: return "out of memory";
        case TC_E_NODEV: return "metadata-only pool has no KV storage";
    }
    return "unknown status";
}

const char *tc_last_error(tc_pool *p) { return p ? p->impl.last_error.c_str() : ""; }

tc_status tc_gather_dev(tc_pool *p, const int32_t *ids, int64_t n, void *dst_dev, void *cuda_stream) {
    TC_GUARD(p) { return P.device_tier(true, ids, n, dst_dev, static_cast<cudaStream_t>(cuda_stream)); }
    TC_CATCH
}

tc_status tc_scatter_dev(tc_pool *p, const void *src_dev, const int32_t *ids, int64_t n, void *cuda_stream) {
    TC_GUARD(p) {
        return P.device_tier(false, ids, n, const_cast<void *>(src_dev), static_cast<cudaStream_t>(cuda_stream));
    }
    TC_CATCH
}

}  // extern "C"
