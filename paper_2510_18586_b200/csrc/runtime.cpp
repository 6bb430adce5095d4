// Host runtime of the Tokencake offload/upload hot path (see runtime.hpp).  Every mutating call validates fully,
// then enqueues GPU work, then commits host state: a non-CUDA error leaves the pool unchanged (strong guarantee).
#include "runtime.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <unordered_set>

namespace tc {

// ------------------------------------------------------------------------------------------------ BlockAllocator
void BlockAllocator::init(int64_t n_blocks, int n_classes) {
    n = n_blocks;
    const int64_t words = (n + 63) / 64;
    bits.assign(words, ~0ull);
    if (n % 64) bits[words - 1] = (1ull << (n % 64)) - 1;
    nfree = n;
    hint = 0;
    state.assign(n, kFree);
    own_agent.assign(n, -1);
    own_pos.assign(n, -1);
    reserved.assign(n_classes, 0);
    claimed.assign(n_classes, 0);
}

int64_t BlockAllocator::unclaimed_sum() const {
    int64_t s = 0;
    for (size_t c = 0; c < reserved.size(); ++c) s += unclaimed((int)c);
    return s;
}

// Reservation first, then shared headroom = free - sum of unclaimed reservations (A9).
int64_t BlockAllocator::plan(int c, int64_t k, int64_t nfree, const std::vector<int64_t> &reserved,
                             const std::vector<int64_t> &claimed) {
    int64_t usum = 0, uc = 0;
    for (size_t x = 0; x < reserved.size(); ++x) {
        const int64_t u = reserved[x] > claimed[x] ? reserved[x] - claimed[x] : 0;
        usum += u;
        if ((int)x == c) uc = u;
    }
    const int64_t r = std::min(k, uc);
    const int64_t s = k - r;
    const int64_t headroom = std::max<int64_t>(0, nfree - usum);
    if (s > headroom || k > nfree) return -1;
    return r;
}

void BlockAllocator::take_lowest(int64_t k, int32_t *out) {
    int64_t got = 0;
    const int64_t words = (int64_t)bits.size();
    for (int64_t w = hint; got < k && w < words; ++w) {
        uint64_t x = bits[w];
        while (x && got < k) {
            const int b = __builtin_ctzll(x);
            out[got++] = (int32_t)(w * 64 + b);
            x &= x - 1;
        }
        bits[w] = x;
    }
    nfree -= got;
    while (hint < words && bits[hint] == 0) ++hint;
}

void BlockAllocator::set_free(int32_t b) {
    bits[b >> 6] |= 1ull << (b & 63);
    ++nfree;
    if ((b >> 6) < hint) hint = b >> 6;
}

// ------------------------------------------------------------------------------------------------ Pool
tc_status Pool::cuda_fail(cudaError_t e, const char *what) {
    cuda_dead = true;
    last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return TC_E_CUDA;
}

#define TC_CUDA(call, what)                                   \
    do {                                                      \
        cudaError_t e__ = (call);                             \
        if (e__ != cudaSuccess) return cuda_fail(e__, what);  \
    } while (0)

static int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

Pool::~Pool() {
    if (meta_only || device < 0) return;
    cudaSetDevice(device);
    if (s_up) cudaStreamSynchronize(s_up);
    if (s_off) cudaStreamSynchronize(s_off);
    for (auto e : events) cudaEventDestroy(e);
    for (auto &sp : spans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
    for (auto e : tev_free) cudaEventDestroy(e);
    if (ev_compute) cudaEventDestroy(ev_compute);
    if (s_up) cudaStreamDestroy(s_up);
    if (s_off) cudaStreamDestroy(s_off);
    if (kv_owned && kv) cudaFree(kv);
    if (table_owned && table_dev) cudaFree(table_dev);
    for (auto st : staging)
        if (st) cudaFree(st);
    if (slots.host) cudaFreeHost(slots.host);
    if (ring_host) cudaFreeHost(ring_host);
}

tc_status Pool::create(const tc_pool_desc &d) {
    if (d.layers < 1 || d.kv_heads < 1 || d.head_dim < 1 || d.block_tokens < 1 || d.n_blocks < 1) return TC_E_INVAL;
    if (d.n_blocks > INT32_MAX - 1) return TC_E_INVAL;
    if (d.dtype != TC_FP16 && d.dtype != TC_BF16) return TC_E_INVAL;
    const int world = d.shard_world < 1 ? 1 : d.shard_world;
    if (d.kv_heads % world || d.shard_rank < 0 || d.shard_rank >= world) return TC_E_INVAL;
    L = d.layers; H = d.kv_heads; D = d.head_dim; T = d.block_tokens; dtype = d.dtype;
    this->world = world; rank = d.shard_rank; Hl = H / world;
    N = d.n_blocks;
    C = (int64_t)T * Hl * D * 2;
    if (C % 16 || (D * 2) % 8) return TC_E_INVAL;   // 16-byte vector path; 8-byte content words per head row
    B = 2 * (int64_t)L * C;
    n_classes = d.n_classes ? d.n_classes : 8;
    if (n_classes < 1 || n_classes > 64) return TC_E_INVAL;
    max_agents = d.max_agents ? d.max_agents : 1024;
    max_bpa = d.max_blocks_per_agent ? d.max_blocks_per_agent : 4096;
    if (max_agents < 1 || max_bpa < 1) return TC_E_INVAL;
    if ((int64_t)max_agents * max_bpa > INT32_MAX) return TC_E_INVAL;
    const int64_t S = d.host_slots > 0 ? d.host_slots : (N * 18 + 99) / 100;
    alloc.init(N, n_classes);
    agents.assign(max_agents, AgentRec{});
    stamp.assign(N, 0);
    slots.count = S;
    slots.slot_bytes = B;
    slots.free_list.resize(S);
    for (int64_t i = 0; i < S; ++i) slots.free_list[i] = S - 1 - i;   // pop() yields 0, 1, 2, ...
    device = d.device;
    meta_only = d.device < 0;
    mode_d2h = d.xfer_d2h;
    mode_h2d = d.xfer_h2d;
    if (mode_d2h < 0 || mode_d2h > 2 || mode_h2d < 0 || mode_h2d > 2) return TC_E_INVAL;
    ctas_d2h = env_int("TC_CTAS_D2H", 0);
    ctas_h2d = env_int("TC_CTAS_H2D", 0);
    ctas_dev = env_int("TC_CTAS_DEV", 0);
    threads = env_int("TC_THREADS", 256);
    if (meta_only) return TC_OK;

    TC_CUDA(cudaSetDevice(device), "cudaSetDevice");
    int lo = 0, hi = 0;
    TC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    TC_CUDA(cudaStreamCreateWithPriority(&s_up, cudaStreamNonBlocking, hi), "upload stream");   // P:646 first
    TC_CUDA(cudaStreamCreateWithPriority(&s_off, cudaStreamNonBlocking, lo), "offload stream");
    TC_CUDA(cudaEventCreateWithFlags(&ev_compute, cudaEventDisableTiming), "event");
    const int64_t kv_bytes = (int64_t)L * 2 * N * C;
    if (d.kv_dev) {
        if (reinterpret_cast<uintptr_t>(d.kv_dev) % 16) return TC_E_INVAL;
        kv = static_cast<char *>(d.kv_dev);
    } else {
        if (cudaMalloc(&kv, kv_bytes) != cudaSuccess) { cudaGetLastError(); kv = nullptr; return TC_E_OOM; }
        kv_owned = true;
    }
    const int64_t tab_bytes = (int64_t)max_agents * max_bpa * 4;
    if (d.table_dev) {
        table_dev = d.table_dev;
    } else {
        if (cudaMalloc(&table_dev, tab_bytes) != cudaSuccess) { cudaGetLastError(); table_dev = nullptr; return TC_E_OOM; }
        table_owned = true;
    }
    TC_CUDA(cudaMemsetAsync(table_dev, 0xFF, tab_bytes, s_off), "table init");
    // CPU block buffer: one pinned, mapped slab allocated once (P:481-484 — no OS alloc/free on the hot path).
    if (cudaHostAlloc(reinterpret_cast<void **>(&slots.host), (size_t)(S * B),
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError(); slots.host = nullptr; return TC_E_OOM;
    }
    TC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&slots.dev), slots.host, 0), "slot dev ptr");
    ring_cap = d.desc_bytes > 0 ? d.desc_bytes : (16ll << 20);
    if (cudaHostAlloc(reinterpret_cast<void **>(&ring_host), (size_t)ring_cap,
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError(); ring_host = nullptr; return TC_E_OOM;
    }
    TC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&ring_dev), ring_host, 0), "ring dev ptr");
    staging_bytes = d.staging_bytes > 0 ? d.staging_bytes : (256ll << 20);
    if (staging_bytes < B) staging_bytes = B;
    if (mode_d2h == TC_XFER_AUTO) mode_d2h = env_int("TC_AUTO_D2H", TC_XFER_DIRECT);
    if (mode_h2d == TC_XFER_AUTO) mode_h2d = env_int("TC_AUTO_H2D", TC_XFER_DIRECT);
    for (int i = 0; i < 16; ++i) {
        cudaEvent_t e;
        TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        events.push_back(e);
        ev_free.push_back(i);
    }
    TC_CUDA(cudaStreamSynchronize(s_off), "create sync");
    return TC_OK;
}

int32_t Pool::event_get() {
    if (ev_free.empty()) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return -1;
        events.push_back(e);
        ev_free.push_back((int32_t)events.size() - 1);
    }
    const int32_t i = ev_free.back();
    ev_free.pop_back();
    ev_used.push_back(i);
    return i;
}

cudaEvent_t Pool::tev_get() {
    if (!tev_free.empty()) {
        cudaEvent_t e = tev_free.back();
        tev_free.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}

tc_status Pool::span_begin(cudaStream_t s, cudaEvent_t *a) {
    *a = nullptr;
    if (!timing) return TC_OK;
    *a = tev_get();
    if (!*a) return cuda_fail(cudaErrorMemoryAllocation, "timing event");
    TC_CUDA(cudaEventRecord(*a, s), "timing event");
    return TC_OK;
}

tc_status Pool::span_end(cudaStream_t s, int32_t kind, cudaEvent_t a, int64_t bytes) {
    if (!timing || !a) return TC_OK;
    cudaEvent_t b = tev_get();
    if (!b) return cuda_fail(cudaErrorMemoryAllocation, "timing event");
    TC_CUDA(cudaEventRecord(b, s), "timing event");
    spans.push_back(Span{kind, a, b, bytes});
    return TC_OK;
}

// Called after both copy streams (and any foreign stream used since) have drained.
void Pool::spans_collect() {
    for (auto &sp : spans) {
        float ms = 0.f;
        if (cudaEventSynchronize(sp.b) == cudaSuccess && cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) {
            tacc.ms[sp.kind] += ms;
            tacc.count[sp.kind] += 1;
            tacc.bytes[sp.kind] += sp.bytes;
        }
        tev_free.push_back(sp.a);
        tev_free.push_back(sp.b);
    }
    spans.clear();
}

// Pinned, mapped scratch for descriptors and table pushes.  Wrapping waits for every stream that may still read it.
char *Pool::ring_alloc(int64_t bytes, char **dev_ptr) {
    bytes = (bytes + 255) & ~255ll;
    if (ring_head + bytes > ring_cap) {
        cudaStreamSynchronize(s_up);
        cudaStreamSynchronize(s_off);
        if (s_compute) cudaStreamSynchronize(s_compute);
        for (cudaStream_t f : foreign) cudaStreamSynchronize(f);
        ring_head = 0;
        if (bytes > ring_cap) {
            cudaFreeHost(ring_host);
            ring_cap = std::max(bytes, ring_cap * 2);
            if (cudaHostAlloc(reinterpret_cast<void **>(&ring_host), (size_t)ring_cap,
                              cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
                ring_host = nullptr;
                return nullptr;
            }
            cudaHostGetDevicePointer(reinterpret_cast<void **>(&ring_dev), ring_host, 0);
        }
    }
    char *h = ring_host + ring_head;
    *dev_ptr = ring_dev + ring_head;
    ring_head += bytes;
    return h;
}

// Enqueue one transfer of desc.size() blocks on stream s.  gather = offload direction (pool -> ext).
// slot_of[i] = host slot of block i (or -1 for the device tier, where desc[i].ext is already set).
tc_status Pool::enqueue_xfer(bool gather, int32_t mode, const std::vector<XferDesc> &desc_in,
                             const std::vector<int64_t> &slot_of, cudaStream_t s) {
    const int64_t n = (int64_t)desc_in.size();
    const XferGeom g{N, C, 2 * L};
    const int ctas = slot_of.empty() ? ctas_dev : (gather ? ctas_d2h : ctas_h2d);
    if (slot_of.empty() || mode == TC_XFER_DIRECT) {
        char *dptr = nullptr;
        char *h = ring_alloc(n * (int64_t)sizeof(XferDesc), &dptr);
        if (!h) return cuda_fail(cudaErrorMemoryAllocation, "descriptor ring");
        XferDesc *hd = reinterpret_cast<XferDesc *>(h);
        for (int64_t i = 0; i < n; ++i) {
            hd[i] = desc_in[i];
            if (!slot_of.empty()) hd[i].ext = reinterpret_cast<uint64_t>(slots.dev + slot_of[i] * B);
        }
        cudaEvent_t t0;
        tc_status st = span_begin(s, &t0);
        if (st != TC_OK) return st;
        TC_CUDA(launch_xfer(gather, reinterpret_cast<const XferDesc *>(dptr), n, g, kv, table_dev, ctas, threads, s),
                "xfer kernel");
        ++n_launch;
        return span_end(s, slot_of.empty() ? 2 : (gather ? 0 : 1), t0, n * B);
    }
    // STAGED: device staging ring + copy-engine DMA over contiguous runs of host slots, in ring-sized pieces.
    char *stg = staging[gather ? 0 : 1];
    if (!stg) {
        TC_CUDA(cudaMalloc(&staging[gather ? 0 : 1], staging_bytes), "staging alloc");
        stg = staging[gather ? 0 : 1];
    }
    const int64_t per = std::max<int64_t>(1, staging_bytes / B);
    for (int64_t a = 0; a < n; a += per) {
        const int64_t b = std::min(n, a + per);
        char *dptr = nullptr;
        char *h = ring_alloc((b - a) * (int64_t)sizeof(XferDesc), &dptr);
        if (!h) return cuda_fail(cudaErrorMemoryAllocation, "descriptor ring");
        XferDesc *hd = reinterpret_cast<XferDesc *>(h);
        for (int64_t i = a; i < b; ++i) {
            hd[i - a] = desc_in[i];
            hd[i - a].ext = reinterpret_cast<uint64_t>(stg + (i - a) * B);
        }
        auto copy_runs = [&](bool to_host) -> tc_status {
            cudaEvent_t t0;
            tc_status st0 = span_begin(s, &t0);
            if (st0 != TC_OK) return st0;
            int64_t i = a;
            while (i < b) {
                int64_t j = i + 1;
                while (j < b && slot_of[j] == slot_of[j - 1] + 1) ++j;
                char *hp = slots.host + slot_of[i] * B;
                char *dp = stg + (i - a) * B;
                TC_CUDA(cudaMemcpyAsync(to_host ? (void *)hp : (void *)dp, to_host ? (void *)dp : (void *)hp,
                                        (size_t)((j - i) * B), to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice,
                                        s),
                        "staged memcpy");
                ++n_memcpy;
                i = j;
            }
            return span_end(s, to_host ? 3 : 4, t0, (b - a) * B);
        };
        cudaEvent_t t0;
        if (gather) {
            tc_status st = span_begin(s, &t0);
            if (st != TC_OK) return st;
            TC_CUDA(launch_xfer(true, reinterpret_cast<const XferDesc *>(dptr), b - a, g, kv, table_dev, ctas_dev,
                                threads, s),
                    "gather kernel");
            ++n_launch;
            st = span_end(s, 0, t0, (b - a) * B);
            if (st != TC_OK) return st;
            st = copy_runs(true);
            if (st != TC_OK) return st;
        } else {
            tc_status st = copy_runs(false);
            if (st != TC_OK) return st;
            st = span_begin(s, &t0);
            if (st != TC_OK) return st;
            TC_CUDA(launch_xfer(false, reinterpret_cast<const XferDesc *>(dptr), b - a, g, kv, table_dev, ctas_dev,
                                threads, s),
                    "scatter kernel");
            ++n_launch;
            st = span_end(s, 1, t0, (b - a) * B);
            if (st != TC_OK) return st;
        }
    }
    return TC_OK;
}

// Device block-table rows follow host-side appends (decode growth) on the stream the agent's compute reads from.
tc_status Pool::table_push(int32_t a, int64_t pos0, int64_t n) {
    if (meta_only) return TC_OK;
    cudaStream_t s = s_compute ? s_compute : s_off;
    AgentRec &ag = agents[a];
    if (ag.up_event >= 0) TC_CUDA(cudaStreamWaitEvent(s, events[ag.up_event], 0), "table push wait");
    char *dptr = nullptr;
    char *h = ring_alloc(n * 4, &dptr);
    if (!h) return cuda_fail(cudaErrorMemoryAllocation, "ring");
    std::memcpy(h, ag.table.data() + pos0, (size_t)n * 4);
    TC_CUDA(cudaMemcpyAsync(table_dev + (int64_t)a * max_bpa + pos0, h, (size_t)n * 4, cudaMemcpyHostToDevice, s),
            "table push");
    ++n_memcpy;
    return TC_OK;
}

// ------------------------------------------------------------------------------------------------ ops
tc_status Pool::reserve(int32_t c, int64_t k) {
    if (c < 0 || c >= n_classes || k < 0) return TC_E_INVAL;
    int64_t total = 0;
    for (int x = 0; x < n_classes; ++x) total += (x == c) ? k : alloc.reserved[x];
    if (total > N) return TC_E_INVAL;
    alloc.reserved[c] = k;            // claimed untouched: lazy shrink
    return TC_OK;
}

tc_status Pool::agent_add(int32_t a, int32_t c) {
    if (a < 0 || a >= max_agents || agents[a].exists || c < 0 || c >= n_classes) return TC_E_INVAL;
    agents[a] = AgentRec{};
    agents[a].exists = true;
    agents[a].cls = c;
    ++n_agents;
    return TC_OK;
}

tc_status Pool::alloc_blocks(int32_t a, int64_t k, int32_t *out) {
    if (cuda_dead) return TC_E_CUDA;
    if (a < 0 || a >= max_agents || !agents[a].exists || k < 1) return TC_E_INVAL;
    AgentRec &ag = agents[a];
    if ((int64_t)ag.table.size() + k > max_bpa) return TC_E_INVAL;
    const int64_t r = BlockAllocator::plan(ag.cls, k, alloc.nfree, alloc.reserved, alloc.claimed);
    if (r < 0) return TC_E_NOBLOCKS;
    const int64_t pos0 = (int64_t)ag.table.size();
    alloc.take_lowest(k, out);
    alloc.claimed[ag.cls] += r;
    for (int64_t i = 0; i < k; ++i) {
        alloc.state[out[i]] = kAlloc;
        alloc.own_agent[out[i]] = a;
        alloc.own_pos[out[i]] = (int32_t)(pos0 + i);
        ag.table.push_back(out[i]);
    }
    return table_push(a, pos0, k);
}

tc_status Pool::agent_free(int32_t a) {
    if (a < 0 || a >= max_agents || !agents[a].exists) return TC_E_INVAL;
    AgentRec &ag = agents[a];
    if (ag.live_offloads > 0) return TC_E_BUSY;
    int64_t k = 0;
    for (int32_t b : ag.table) {
        if (b < 0) continue;
        alloc.state[b] = kFree;
        alloc.own_agent[b] = -1;
        alloc.own_pos[b] = -1;
        alloc.set_free(b);
        ++k;
    }
    alloc.claimed[ag.cls] -= std::min(k, alloc.claimed[ag.cls]);    // reservation-first return
    ag.table.clear();
    return TC_OK;
}

tc_status Pool::offload_batch(int32_t na, const int32_t *ags, const int64_t *off, const int32_t *ids,
                              tc_handle *out) {
    if (cuda_dead) return TC_E_CUDA;
    if (na < 1 || !ags || !off || !ids || !out || off[0] != 0) return TC_E_INVAL;
    // a2 admission: validate everything before touching state (A5, A15), item by item in order so that the first
    // failing item decides the status (sequential-composition semantics of a batch)
    if (++epoch == 0) { std::fill(stamp.begin(), stamp.end(), 0); epoch = 1; }
    for (int32_t k = 0; k < na; ++k) {
        const int32_t a = ags[k];
        if (a < 0 || a >= max_agents || !agents[a].exists) return TC_E_INVAL;
        if (off[k + 1] - off[k] < 1) return TC_E_INVAL;
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            const int32_t b = ids[i];
            if (b < 0 || b >= N || alloc.state[b] != kAlloc || alloc.own_agent[b] != a || stamp[b] == epoch)
                return TC_E_INVAL;
            stamp[b] = epoch;
        }
        if ((int64_t)slots.free_list.size() < off[k + 1]) return TC_E_NOHOST;   // refuse
    }
    const int64_t n = off[na];

    std::vector<XferDesc> desc(n);
    std::vector<int64_t> slot_of(n);
    const size_t top = slots.free_list.size();
    for (int64_t i = 0; i < n; ++i) slot_of[i] = slots.free_list[top - 1 - i];   // LIFO pop order
    for (int32_t k = 0; k < na; ++k)
        for (int64_t i = off[k]; i < off[k + 1]; ++i)
            desc[i] = XferDesc{ids[i], ags[k] * max_bpa + alloc.own_pos[ids[i]], 0};

    int32_t ev = -1;
    if (!meta_only) {
        if (s_compute) {   // capture the agents' last decode writes (GPU-side, no host block)
            TC_CUDA(cudaEventRecord(ev_compute, s_compute), "compute event");
            TC_CUDA(cudaStreamWaitEvent(s_off, ev_compute, 0), "compute wait");
        }
        for (int32_t k = 0; k < na; ++k) {   // blocks still being written by an upload of this agent
            const int32_t ue = agents[ags[k]].up_event;
            if (ue >= 0) TC_CUDA(cudaStreamWaitEvent(s_off, events[ue], 0), "upload->offload wait");
        }
        tc_status st = enqueue_xfer(true, mode_d2h, desc, slot_of, s_off);
        if (st != TC_OK) return st;
        ev = event_get();
        if (ev < 0) return cuda_fail(cudaErrorMemoryAllocation, "event pool");
        TC_CUDA(cudaEventRecord(events[ev], s_off), "offload event");
        bytes_d2h += n * B;
    }
    // commit (a3 logical effects + a4 pending free)
    slots.free_list.resize(top - n);
    for (int32_t k = 0; k < na; ++k) {
        const int32_t a = ags[k];
        AgentRec &ag = agents[a];
        HandleRec hr;
        hr.agent = a;
        hr.cls = ag.cls;
        hr.state = kOffloaded;
        hr.ev = ev;
        std::vector<int32_t> pend;
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            const int32_t b = ids[i];
            const int32_t p = alloc.own_pos[b];
            hr.pos.push_back(p);
            hr.slots.push_back(slot_of[i]);
            ag.table[p] = -1;
            alloc.state[b] = kPending;
            alloc.own_agent[b] = -1;
            alloc.own_pos[b] = -1;
            pend.push_back(b);
        }
        pending_dev.emplace_back(ag.cls, std::move(pend));
        ++ag.live_offloads;
        const tc_handle h = next_handle++;
        handles.emplace(h, std::move(hr));
        out[k] = h;
    }
    return TC_OK;
}

tc_status Pool::upload_batch(int32_t nh, const tc_handle *hs, const int64_t *off, int32_t *out_ids) {
    if (cuda_dead) return TC_E_CUDA;
    if (nh < 1 || !hs || !off || !out_ids || off[0] != 0) return TC_E_INVAL;
    std::vector<HandleRec *> hr(nh);
    // validate + a5 dry run on counters only, item by item in order (first failing item decides the status)
    std::vector<int64_t> cl = alloc.claimed;
    std::vector<int64_t> rr(nh);
    int64_t nf = alloc.nfree;
    std::unordered_set<tc_handle> seen;
    for (int32_t k = 0; k < nh; ++k) {
        auto it = handles.find(hs[k]);
        if (it == handles.end() || it->second.state != kOffloaded || !seen.insert(hs[k]).second) return TC_E_HANDLE;
        hr[k] = &it->second;
        const int64_t k_n = off[k + 1] - off[k];
        if (k_n != (int64_t)hr[k]->pos.size()) return TC_E_INVAL;
        const int64_t r = BlockAllocator::plan(hr[k]->cls, k_n, nf, alloc.reserved, cl);
        if (r < 0) return TC_E_NOBLOCKS;      // upload "stalls"; handles stay valid
        rr[k] = r;
        cl[hr[k]->cls] += r;
        nf -= k_n;
    }
    const int64_t n = off[nh];
    // sequential composition of lowest-free-first == the n lowest free ids split in order
    std::vector<int32_t> fresh(n);
    {
        int64_t got = 0;
        for (int64_t w = alloc.hint; got < n && w < (int64_t)alloc.bits.size(); ++w)
            for (uint64_t x = alloc.bits[w]; x && got < n; x &= x - 1) fresh[got++] = (int32_t)(w * 64 + __builtin_ctzll(x));
    }
    std::vector<XferDesc> desc(n);
    std::vector<int64_t> slot_of(n);
    for (int32_t k = 0; k < nh; ++k)
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            const int64_t q = i - off[k];
            desc[i] = XferDesc{fresh[i], hr[k]->agent * max_bpa + hr[k]->pos[q], 0};
            slot_of[i] = hr[k]->slots[q];
        }
    int32_t ev = -1;
    if (!meta_only) {
        for (int32_t k = 0; k < nh; ++k)      // A13: the upload waits for the handle's offload (GPU-side)
            if (hr[k]->ev >= 0) TC_CUDA(cudaStreamWaitEvent(s_up, events[hr[k]->ev], 0), "offload->upload wait");
        tc_status st = enqueue_xfer(false, mode_h2d, desc, slot_of, s_up);
        if (st != TC_OK) return st;
        ev = event_get();
        if (ev < 0) return cuda_fail(cudaErrorMemoryAllocation, "event pool");
        TC_CUDA(cudaEventRecord(events[ev], s_up), "upload event");
        bytes_h2d += n * B;
    }
    // commit (a5 allocation, a6 remap, a7 released slots)
    {
        std::vector<int32_t> taken(n);
        alloc.take_lowest(n, taken.data());   // identical to `fresh` (same scan, nothing changed in between)
    }
    for (int32_t k = 0; k < nh; ++k) {
        HandleRec &h = *hr[k];
        AgentRec &ag = agents[h.agent];
        alloc.claimed[h.cls] += rr[k];
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            const int64_t q = i - off[k];
            const int32_t b = fresh[i];
            alloc.state[b] = kAlloc;
            alloc.own_agent[b] = h.agent;
            alloc.own_pos[b] = h.pos[q];
            ag.table[h.pos[q]] = b;
            slots.released.push_back(h.slots[q]);
            out_ids[i] = b;
        }
        h.state = kUploaded;
        h.ev = ev;
        --ag.live_offloads;
        ag.up_event = ev;
    }
    return TC_OK;
}

tc_status Pool::query(tc_handle h, bool wait) {
    auto it = handles.find(h);
    if (it == handles.end()) return TC_E_HANDLE;
    if (meta_only || it->second.ev < 0) return TC_OK;
    cudaEvent_t e = events[it->second.ev];
    if (wait) {
        TC_CUDA(cudaEventSynchronize(e), "wait");
        return TC_OK;
    }
    const cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return TC_OK;
    if (r == cudaErrorNotReady) return TC_E_BUSY;
    return cuda_fail(r, "query");
}

tc_status Pool::stream_wait(tc_handle h, cudaStream_t s) {
    auto it = handles.find(h);
    if (it == handles.end()) return TC_E_HANDLE;
    if (meta_only || it->second.ev < 0) return TC_OK;
    TC_CUDA(cudaStreamWaitEvent(s, events[it->second.ev], 0), "stream wait");
    return TC_OK;
}

tc_status Pool::sync() {
    if (!meta_only) {
        if (cuda_dead) return TC_E_CUDA;
        TC_CUDA(cudaStreamSynchronize(s_up), "sync upload stream");
        TC_CUDA(cudaStreamSynchronize(s_off), "sync offload stream");
        for (cudaStream_t f : foreign) TC_CUDA(cudaStreamSynchronize(f), "sync caller stream");
        spans_collect();
    }
    for (auto &pc : pending_dev) {        // a4 retire in issue order (A10)
        for (int32_t b : pc.second) {
            alloc.state[b] = kFree;
            alloc.set_free(b);
        }
        const int64_t k = (int64_t)pc.second.size();
        alloc.claimed[pc.first] -= std::min(k, alloc.claimed[pc.first]);
    }
    pending_dev.clear();
    // released host slots back to the buffer; pushed in reverse so later pops replay ascending runs
    for (auto it = slots.released.rbegin(); it != slots.released.rend(); ++it) slots.free_list.push_back(*it);
    slots.released.clear();
    for (auto it = handles.begin(); it != handles.end();) {
        if (it->second.state == kUploaded) {
            it = handles.erase(it);
        } else {
            it->second.ev = -1;
            ++it;
        }
    }
    for (auto &ag : agents) ag.up_event = -1;
    for (int32_t e : ev_used) ev_free.push_back(e);
    ev_used.clear();
    return TC_OK;
}

tc_status Pool::fill(uint64_t seed) {
    if (meta_only) return TC_E_NODEV;
    if (cuda_dead) return TC_E_CUDA;
    TC_CUDA(launch_fill(kv, N, L, T, H, Hl, rank, D, seed, s_off), "fill kernel");
    ++n_launch;
    TC_CUDA(cudaStreamSynchronize(s_off), "fill sync");
    return TC_OK;
}

tc_status Pool::device_tier(bool gather, const int32_t *ids, int64_t n, void *ext, cudaStream_t s) {
    if (meta_only) return TC_E_NODEV;
    if (cuda_dead) return TC_E_CUDA;
    if (n < 1 || !ids || !ext || reinterpret_cast<uintptr_t>(ext) % 16) return TC_E_INVAL;
    std::vector<XferDesc> desc(n);
    for (int64_t i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= N) return TC_E_INVAL;
        desc[i] = XferDesc{ids[i], -1, reinterpret_cast<uint64_t>(static_cast<char *>(ext) + i * B)};
    }
    if (s && s != s_off && s != s_up && s != s_compute &&
        std::find(foreign.begin(), foreign.end(), s) == foreign.end())
        foreign.push_back(s);   // ring wrap must also wait for descriptor reads on caller streams
    return enqueue_xfer(gather, TC_XFER_DIRECT, desc, {}, s ? s : s_off);
}

}  // namespace tc
