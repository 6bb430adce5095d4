// Host runtime of the Tokencake offload/upload hot path (see runtime.hpp).  Every mutating call validates fully,
// then enqueues GPU work, then commits host state: a non-CUDA error leaves the pool unchanged (strong guarantee).
#include "runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
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

// ------------------------------------------------------------------------------------------------ HostSlots
void HostSlots::init(int64_t S) {
    count = S;
    const int64_t words = (S + 63) / 64;
    bits.assign(words, ~0ull);
    if (S % 64) bits[words - 1] = (1ull << (S % 64)) - 1;
    nfree = S;
}

void HostSlots::choose(int64_t n, int64_t *out) const {
    if (n <= 0) return;
    int64_t start = 0, len = 0;
    for (size_t w = 0; w < bits.size(); ++w) {
        const uint64_t x = bits[w];
        if (x == ~0ull) {                                  // a whole free word extends the run
            if (len == 0) start = (int64_t)w * 64;
            len += 64;
            if (len >= n) break;
            continue;
        }
        if (x == 0) {
            len = 0;
            continue;
        }
        for (int b = 0; b < 64; ++b) {
            if ((x >> b) & 1) {
                if (len == 0) start = (int64_t)w * 64 + b;
                if (++len >= n) break;
            } else {
                len = 0;
            }
        }
        if (len >= n) break;
    }
    if (len >= n) {
        for (int64_t i = 0; i < n; ++i) out[i] = start + i;
        return;
    }
    int64_t got = 0;                                       // fragmented: the lowest free slots
    for (size_t w = 0; w < bits.size() && got < n; ++w)
        for (uint64_t x = bits[w]; x && got < n; x &= x - 1) out[got++] = (int64_t)w * 64 + __builtin_ctzll(x);
}

void HostSlots::take(const int64_t *s, int64_t n) {
    for (int64_t i = 0; i < n; ++i) bits[s[i] >> 6] &= ~(1ull << (s[i] & 63));
    nfree -= n;
}

static int64_t steady_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// ------------------------------------------------------------------------------------------------ host trace
// TC_HOST_TRACE=1: per tc_cycle, the host time (µs from the call's entry) at which each enqueue step returned, on
// stderr.  A debugging aid for the enqueue critical path (how soon each link direction gets its first DMA).
static bool g_trace = std::getenv("TC_HOST_TRACE") != nullptr;
static std::chrono::steady_clock::time_point g_trace_t0;
static std::string g_trace_buf;
static void trace(const char *what) {
    if (!g_trace) return;
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - g_trace_t0).count();
    char b[96];
    std::snprintf(b, sizeof b, " %s=%.1f", what, us);
    g_trace_buf += b;
}

// ------------------------------------------------------------------------------------------------ Pool
// A host allocation failed after part of a batch's GPU work was enqueued: the device may already be rewriting the
// table / pool for a batch the host never committed, so the pool is poisoned like on a CUDA error (TC_E_OOM, then
// TC_E_CUDA for every later call).  Allocation failures before the enqueue (plan_*) leave the pool unchanged.
tc_status Pool::enqueue_oom() {
    cuda_dead = true;
    last_error = "host allocation failed while enqueueing a transfer (pool poisoned)";
    return TC_E_OOM;
}

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
    for (auto e : fev_live) cudaEventDestroy(e);
    for (auto &ag : agents)
        if (ag.push_ev) cudaEventDestroy(ag.push_ev);
    for (auto e : fev_free) cudaEventDestroy(e);
    for (auto &d2 : half_free)
        for (auto e : d2)
            if (e) cudaEventDestroy(e);
    if (s_up) cudaStreamDestroy(s_up);
    if (s_up_k) cudaStreamDestroy(s_up_k);
    if (s_off_k) cudaStreamDestroy(s_off_k);
    if (s_off) cudaStreamDestroy(s_off);
    if (kv_owned && kv) cudaFree(kv);
    if (table_owned && table_dev) cudaFree(table_dev);
    for (auto st : staging)
        if (st) cudaFree(st);
    if (slots.host) cudaFreeHost(slots.host);
    for (auto &kv_ : extra)
        if (kv_.second.host) cudaFreeHost(kv_.second.host);
    if (ring_host) cudaFreeHost(ring_host);
    if (kts_dev) cudaFree(kts_dev);
    if (peer.dev) cudaFree(peer.dev);
}

tc_status Pool::create(const tc_pool_desc &d) {
    if (d.layers < 1 || d.kv_heads < 1 || d.head_dim < 1 || d.block_tokens < 1 || d.n_blocks < 1) return TC_E_INVAL;
    if (d.n_blocks > INT32_MAX - 1) return TC_E_INVAL;
    if (d.dtype != TC_FP16 && d.dtype != TC_BF16) return TC_E_INVAL;
    const int g = d.shard_world < 1 ? 1 : d.shard_world;
    if (d.kv_heads % g || d.shard_rank < 0 || d.shard_rank >= g) return TC_E_INVAL;
    L = d.layers; H = d.kv_heads; D = d.head_dim; T = d.block_tokens; dtype = d.dtype;
    world = g; rank = d.shard_rank; Hl = H / g;
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
    slots.init(S);
    slots.slot_bytes = B;
    device = d.device;
    meta_only = d.device < 0;
    check = env_int("TC_CHECK", 0) != 0;
    fine_off = env_int("TC_FINE_DEPS", 1) == 0;
    min_piece_bytes = env_int("TC_MIN_PIECE_MIB", 64) * (1ll << 20);
    unbuffered = d.unbuffered != 0;
    next_slot = S;
    mode_d2h = d.xfer_d2h;
    mode_h2d = d.xfer_h2d;
    if (mode_d2h < 0 || mode_d2h > 3 || mode_h2d < 0 || mode_h2d > 3) return TC_E_INVAL;
    // NEXT-2 peer tier (reading C1): slot ids S .. S+P-1, own LIFO free list (pops ascending)
    if (d.peer_slots < 0 || (d.peer_slots > 0 && unbuffered)) return TC_E_INVAL;
    peer.count = d.peer_slots;
    peer.device = d.peer_device;
    peer.free_list.resize(peer.count);
    for (int64_t i = 0; i < peer.count; ++i) peer.free_list[i] = S + peer.count - 1 - i;
    // Default launch configuration per path: TMA bulk everywhere.  The DIRECT kernels move bytes over
    // the host link for the whole transfer, so they get a fixed small grid — 32 CTAs for the mapped-host writes
    // (D2H), 74 for the reads (H2D) — that leaves the other direction's kernel and the engine's compute room on the
    // SMs; the old 592 x 256-thread SIMT grid filled every register file, so a concurrent D2H and H2D ran one after
    // the other (profiles/r02_direct_probe_c2_*.json).  Device side / peer tier: the size-adaptive grid (0).
    const char *path_names[4] = {"D2H", "H2D", "DEV", "PEER"};
    const int default_ctas[4] = {32, 74, 0, 0};
    for (int i = 0; i < 4; ++i) {
        char nm[32];
        std::snprintf(nm, sizeof nm, "TC_CTAS_%s", path_names[i]);
        ctas[i] = env_int(nm, default_ctas[i]);
        std::snprintf(nm, sizeof nm, "TC_THREADS_%s", path_names[i]);
        nthreads[i] = env_int(nm, 256);
        std::snprintf(nm, sizeof nm, "TC_VARIANT_%s", path_names[i]);
        variant[i] = env_int(nm, 3);
    }
    if (meta_only) return TC_OK;

    TC_CUDA(cudaSetDevice(device), "cudaSetDevice");
    int lo = 0, hi = 0;
    TC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    // TC_UP_PRIORITY=0: the upload streams at the default priority too (A/B of the copy-engine behaviour)
    const int up_prio = env_int("TC_UP_PRIORITY", 1) ? hi : lo;
    TC_CUDA(cudaStreamCreateWithPriority(&s_up, cudaStreamNonBlocking, up_prio), "upload stream");   // P:646 first
    TC_CUDA(cudaStreamCreateWithPriority(&s_off, cudaStreamNonBlocking, lo), "offload stream");
    TC_CUDA(cudaStreamCreateWithPriority(&s_up_k, cudaStreamNonBlocking, up_prio), "upload aux stream");
    TC_CUDA(cudaStreamCreateWithPriority(&s_off_k, cudaStreamNonBlocking, lo), "offload aux stream");
    piece_bytes = env_int("TC_PIECE_KIB", 256 * 1024) * 1024ll;
    head_bytes = env_int("TC_HEAD_KIB", 0) * 1024ll;
    halves = env_int("TC_STAGING_HALVES", 1) != 0;
    TC_CUDA(cudaEventCreateWithFlags(&ev_compute, cudaEventDisableTiming), "event");
    for (auto &d2 : half_free)
        for (auto &e : d2) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
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
    if (peer.count > 0) {                     // the peer slab lives in the neighbour's HBM, reached over NVLink
        if (peer.device < 0) return TC_E_INVAL;
        if (peer.device != device) {
            int ok = 0;
            TC_CUDA(cudaDeviceCanAccessPeer(&ok, device, peer.device), "peer query");
            if (!ok) return TC_E_INVAL;
            const cudaError_t e = cudaDeviceEnablePeerAccess(peer.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "enable peer access");
            cudaGetLastError();
            TC_CUDA(cudaSetDevice(peer.device), "cudaSetDevice(peer)");
        }
        const cudaError_t e = cudaMalloc(&peer.dev, (size_t)(peer.count * B));
        cudaSetDevice(device);
        if (e != cudaSuccess) { cudaGetLastError(); peer.dev = nullptr; return TC_E_OOM; }
    }
    staging_bytes = d.staging_bytes > 0 ? d.staging_bytes : env_int("TC_STAGING_MIB", 1024) * (1ll << 20);
    // at least two blocks: a batch larger than the buffer alternates two halves of >= 1 block each (xfer_base)
    if (staging_bytes < 2 * B) staging_bytes = 2 * B;
    // AUTO: the copy-engine staged path measured fastest for full cycles on B200 (profiles/r01_staged_ab.md).
    auto_dir[0] = mode_d2h == TC_XFER_AUTO;
    auto_dir[1] = mode_h2d == TC_XFER_AUTO;
    auto_choice[0] = env_int("TC_AUTO_D2H", TC_XFER_STAGED);
    auto_choice[1] = env_int("TC_AUTO_H2D", TC_XFER_STAGED);
    if (auto_dir[0]) mode_d2h = auto_mode(0);
    if (auto_dir[1]) mode_h2d = auto_mode(1);
    auto_direct_bytes[0] = auto_direct_bytes[1] = env_int("TC_AUTO_DIRECT_KIB", 2048) * 1024ll;
    // completion events, created up front (a deep retire lag keeps dozens in flight; no driver call inside a loop)
    for (int i = 0; i < 256; ++i) {
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
    if ((size_t)i >= ev_epoch.size()) ev_epoch.resize(events.size(), 0);
    ev_epoch[i] = epoch_id;
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

// Event spans: timing 1 around every kernel launch and DMA run; timing 3 around kernel launches only (the DMAs keep
// their schedule untouched; the kernels are also stamped, as in 2).
bool Pool::span_on(bool kernel) const { return timing == 1 || (timing == 3 && kernel); }

tc_status Pool::span_begin(cudaStream_t s, cudaEvent_t *a, bool kernel) {
    *a = nullptr;
    if (!span_on(kernel)) return TC_OK;
    *a = tev_get();
    if (!*a) return cuda_fail(cudaErrorMemoryAllocation, "timing event");
    TC_CUDA(cudaEventRecord(*a, s), "timing event");
    return TC_OK;
}

tc_status Pool::span_end(cudaStream_t s, int32_t kind, cudaEvent_t a, int64_t bytes, bool link) {
    if (!a) return TC_OK;
    cudaEvent_t b = tev_get();
    if (!b) return cuda_fail(cudaErrorMemoryAllocation, "timing event");
    TC_CUDA(cudaEventRecord(b, s), "timing event");
    spans.push_back(Span{kind, a, b, bytes, link && kind != 2});
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
            if (sp.link && B > 0) {                             // the host-link side of a transfer
                const int dir = (sp.kind == 7 || sp.kind == 3) ? 0 : 1;
                const double nb = (double)(sp.bytes / B);
                cal_ms[dir] += ms;
                cal_blocks[dir] += sp.bytes / B;
                cal_cnt[dir] += 1;
                cal_nn[dir] += nb * nb;
                cal_nt[dir] += nb * ms;
            }
            if (timeline.size() < (size_t)timeline_cap) {      // start/end relative to this sync interval's first span
                float t0 = 0.f;
                cudaEventElapsedTime(&t0, spans.front().a, sp.a);
                timeline.push_back(tc_span_t{sync_count, sp.kind, (double)t0, (double)(t0 + ms), sp.bytes});
            }
        }
        tev_free.push_back(sp.a);
        tev_free.push_back(sp.b);
    }
    spans.clear();
}

// Device-side kernel durations (%globaltimer stamps) of the launches since the last collection.  Deferred: called by
// tc_timing() and by tc_sync only when the stamp buffer is nearly full, so a sync costs no extra copies while
// timing mode 2 runs (the bench's timed region).  Callers have drained the streams.
void Pool::stamps_collect() {
    if (!kts_meta.empty()) {
        const size_t used = kts_meta.size();
        std::vector<unsigned long long> buf(2 * used);
        if (cudaMemcpy(buf.data(), kts_dev, used * 16, cudaMemcpyDeviceToHost) == cudaSuccess) {
            // TC_STAMP_DUMP=FILE (diagnostics): append "kind start_ns end_ns bytes" per launch
            static const char *dump = std::getenv("TC_STAMP_DUMP");
            if (dump) {
                if (FILE *f = std::fopen(dump, "a")) {
                    for (size_t i = 0; i < used; ++i)
                        std::fprintf(f, "%d %llu %llu %lld\n", kts_meta[i].first, buf[2 * i], buf[2 * i + 1],
                                     (long long)kts_meta[i].second);
                    std::fclose(f);
                }
            }
            for (size_t i = 0; i < used; ++i) {
                if (buf[2 * i + 1] < buf[2 * i]) continue;          // launch had no CTA with work
                const int k = kts_meta[i].first;
                tacc.kernel_ms[k] += (double)(buf[2 * i + 1] - buf[2 * i]) * 1e-6;
                tacc.kernel_count[k] += 1;
                tacc.kernel_bytes[k] += kts_meta[i].second;
            }
            cudaMemcpy(kts_dev, kts_init.data(), used * 16, cudaMemcpyHostToDevice);
        } else {
            cudaGetLastError();
        }
        kts_meta.clear();
    }
}

// Kernel geometry for one launch; with tc_timing on, also a {start, end} %globaltimer slot for that launch.
// The stamp buffer, allocated when timing is switched on (tc_timing), never inside a timed loop: a cudaMalloc there
// can wait on the driver for tens of milliseconds.
bool Pool::kts_ensure() {
    if (kts_dev) return true;
    if (cudaMalloc(&kts_dev, (size_t)kKts * 16) != cudaSuccess) { cudaGetLastError(); kts_dev = nullptr; return false; }
    kts_init.assign(2 * kKts, 0);
    for (int64_t i = 0; i < kKts; ++i) kts_init[2 * i] = ~0ull;
    if (cudaMemcpy(kts_dev, kts_init.data(), (size_t)kKts * 16, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(kts_dev);
        kts_dev = nullptr;
        return false;
    }
    return true;
}

XferGeom Pool::geom(int32_t kind, int64_t bytes) {
    XferGeom g{N, C, 2 * L, nullptr};
    if (!timing || meta_only) return g;
    if (!kts_ensure()) return g;
    if ((int64_t)kts_meta.size() >= kKts) return g;      // more launches than slots before a sync: untimed
    g.ts = kts_dev + 2 * kts_meta.size();
    kts_meta.emplace_back(kind, bytes);
    return g;
}

char *Pool::host_ptr(int64_t slot) const {
    if (slot < slots.count) return slots.host + slot * B;
    auto sl = std::prev(extra.upper_bound(slot));
    return sl->second.host + (slot - sl->first) * B;
}

char *Pool::host_dev_ptr(int64_t slot) const {
    if (slot < slots.count) return slots.dev + slot * B;
    auto sl = std::prev(extra.upper_bound(slot));
    return sl->second.dev + (slot - sl->first) * B;
}

// Pinned, mapped scratch for descriptors and table pushes.  Wrapping waits for every stream that may still read it.
char *Pool::ring_alloc(int64_t bytes, char **dev_ptr) {
    bytes = (bytes + 255) & ~255ll;
    if (ring_head + bytes > ring_cap) {
        cudaStreamSynchronize(s_up);
        cudaStreamSynchronize(s_off);
        if (s_compute) cudaStreamSynchronize(s_compute);
        drain_foreign();
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

// A transfer of desc.size() blocks, enqueued in two phases so that one scheduling cycle can interleave its two
// directions on the host (tc_cycle) and both links start as early as possible:
//   DIRECT          A = the single kernel over mapped host memory                 B = -
//   COPY            A = table kernel (offload) + one strided DMA per block + table kernel (upload)
//   STAGED gather   A = per piece: gather kernel, D2H copy                        B = -
//   STAGED scatter  A = the H2D copy per piece                                    B = the scatter per piece, join
// A staged batch that fits the staging buffer is cut into pieces of piece_bytes (default: one piece).  One piece runs
// kernel and DMA in stream order on the direction's main stream; several pieces pipeline the device-side kernels on
// an aux stream against the copy engine.  TC_HEAD_KIB > 0 adds a small first (gather) / last (scatter) piece, so the
// D2H link starts after a short gather and little scatter trails the last H2D byte — measured slower on B200 than
// one large piece, because every extra DMA and cross-stream hop costs tens of µs (profiles/r01_staged_ab.md).  A
// batch larger than the staging buffer runs double-buffered pieces of half the buffer, issued interleaved in phase
// A (B does nothing).
tc_status Pool::xfer_init(XferJob &j, bool gather, int32_t mode, const std::vector<XferDesc> *desc,
                          const std::vector<int64_t> *slot_of, cudaStream_t s, const int64_t *item_off,
                          int32_t n_items) {
    j.gather = gather;
    j.mode = (slot_of == nullptr || slot_of->empty()) ? TC_XFER_DIRECT : mode;
    j.desc = desc;
    j.slot_of = slot_of;
    j.s = s;
    j.n = (int64_t)desc->size();
    if (j.mode == TC_XFER_STAGED && auto_dir[gather ? 0 : 1] && j.n * B <= auto_direct_bytes[gather ? 0 : 1])
        j.mode = TC_XFER_DIRECT;
    if (j.mode != TC_XFER_STAGED || j.n == 0) return TC_OK;
    const int dir = gather ? 0 : 1;
    if (!staging[dir]) TC_CUDA(cudaMalloc(&staging[dir], staging_bytes), "staging alloc");
    j.stg = staging[dir];
    j.sk = gather ? s_off_k : s_up_k;
    j.cut.clear();
    const int64_t cap = staging_bytes / B;                       // blocks the staging buffer holds (>= 2)
    j.ring_reuse = j.n > cap;
    const int64_t edge = head_bytes > 0 ? std::max<int64_t>(1, head_bytes / B) : 0;   // head / tail blocks
    const int64_t big = std::max<int64_t>(1, piece_bytes / B);
    // With the items' block offsets (a batch of several agents / handles, fine-grained dependencies on), a piece
    // ends on the last item boundary inside its size limit when that leaves it at least min_piece_bytes: an item's
    // last block then lands with its own piece instead of with the next item's first blocks, so its per-handle
    // completion (below) comes sooner.  Ids and bytes do not depend on the cuts.
    const bool align = item_off && n_items > 0 && !fine_off;
    const int64_t min_blocks = std::max<int64_t>(1, min_piece_bytes / B);
    auto cut_by = [&](int64_t step) {
        for (int64_t a = 0; a < j.n;) {
            j.cut.push_back(a);
            int64_t e = std::min(j.n, a + step);
            if (align && e < j.n) {
                const int64_t *q = std::upper_bound(item_off, item_off + n_items + 1, e) - 1;   // last end <= e
                if (*q > a && *q - a >= min_blocks) e = *q;
            }
            a = e;
        }
    };
    if (j.ring_reuse) {
        j.pb = std::max<int64_t>(1, cap / 2);
        cut_by(j.pb);
    } else if (edge == 0) {
        cut_by(big);
    } else if (gather) {
        j.cut.push_back(0);
        for (int64_t a = std::min(edge, j.n); a < j.n; a += big) j.cut.push_back(a);
    } else {
        const int64_t body = std::max<int64_t>(0, j.n - edge);
        for (int64_t a = 0; a < body; a += big) j.cut.push_back(a);
        j.cut.push_back(body);
    }
    j.cut.push_back(j.n);
    j.npieces = (int64_t)j.cut.size() - 1;
    j.ev.assign(j.npieces, -1);
    const int64_t half_bytes = (staging_bytes / 2) & ~255ll;  // half 1 starts 256-byte aligned (TMA needs 16)
    if (j.npieces == 1 && halves && j.n * B <= half_bytes) {
        // one piece that fits half the buffer: alternate halves across batches.  Gather: kernel on the aux stream,
        // D2H on the main stream; upload: H2D on the aux stream, scatter (+ remap, completion) on the main stream.
        // Each waits only for the previous use of its own half, so batch k's kernel overlaps batch k-1's DMA and
        // the copy engine runs the direction's batches back to back.  The caller's GPU-side dependencies (offload
        // / upload waits) are also placed on the aux stream (offload_waits / upload_waits).
        j.half = half_next[dir];
        half_next[dir] ^= 1;
        j.stg = staging[dir] + (int64_t)j.half * half_bytes;
        if (!gather) std::swap(j.s, j.sk);          // DMA stream = aux, kernel stream = main
        TC_CUDA(cudaStreamWaitEvent(gather ? j.sk : j.s, half_free[dir][j.half], 0), "half reuse");
        return TC_OK;
    }
    if (j.npieces == 1) {                            // one piece: kernel and DMA in stream order, no cross-stream hop
        j.sk = j.s;
        return TC_OK;
    }
    j.need_hop = true;                               // phase A: the aux stream starts after the main stream's waits
    return TC_OK;
}

// Fine-grained dependencies: the items (one agent's offload, one handle's upload) held by blocks [a, b) of the job.
tc_status Pool::piece_waits(const XferJob &j, int64_t a, int64_t b, cudaStream_t st) {
    if (!j.item_dep) return TC_OK;
    int64_t k = std::upper_bound(j.item_off, j.item_off + j.n_items + 1, a) - j.item_off - 1;
    int32_t last = -1;
    for (; k < j.n_items && j.item_off[k] < b; ++k) {
        const int32_t e = j.item_dep[k];
        if (e >= 0 && e != last) TC_CUDA(cudaStreamWaitEvent(st, events[e], 0), "item wait");
        if (e >= 0) last = e;
    }
    return TC_OK;
}

// A staged job of several pieces waits per piece for the items it holds and marks each piece's end, so a batch's
// first items do not wait for its last items' dependencies, and a handle completes with the piece holding its last
// block instead of with the whole batch (a cycle's uploads can start on the first offloads of the previous cycle
// as soon as their pieces are on the host).  Ordering only: ids and bytes are unchanged.
bool Pool::fine_grained(XferJob &j, const int64_t *item_off, int32_t n_items, const std::vector<int32_t> &deps) {
    if (j.mode != TC_XFER_STAGED || j.npieces < 2 || fine_off) return false;
    j.item_off = item_off;
    j.item_dep = deps.data();
    j.n_items = n_items;
    j.piece_done.assign(j.npieces, -1);
    return true;
}

// Per-item completion events of a fine-grained job: the piece holding the item's last block.
void Pool::item_events(const XferJob &j, std::vector<int32_t> &out) const {
    out.resize(j.n_items);
    for (int32_t k = 0; k < j.n_items; ++k) {
        const int64_t last = j.item_off[k + 1] - 1;
        const int64_t p = std::upper_bound(j.cut.begin(), j.cut.end(), last) - j.cut.begin() - 1;
        out[k] = j.piece_done[p];
    }
}

// AUTO: the path measured fastest for a full scheduling cycle on B200 (both directions concurrently).
// A batch of at most auto_direct_bytes[dir] still takes the DIRECT kernel: one launch instead of kernel + DMA, ~5 µs
// sooner for 1-2 blocks and equal from ~2 MiB up (profiles/r01_sweep_c{2,5}.json); tc_calibrate re-measures the
// crossover per direction on the box (calibrate_small).
int32_t Pool::auto_mode(int dir) const { return auto_choice[dir]; }

// The small-batch crossover (north_star: DIRECT "chosen against a device-staging path ... according to the measured
// bandwidth"): one direction alone, batches of 1, 2, 4, ... blocks, DIRECT vs STAGED completion time (best of 5 after
// a warm-up); auto_direct_bytes[dir] = the largest size up to which DIRECT was never slower.  Same blocks and slots as
// calibrate's probe, so the pool's contents stay unchanged (gathers only read; scatters rewrite B's own bytes).
tc_status Pool::calibrate_small(int64_t k, const std::vector<XferDesc> &da, const std::vector<XferDesc> &db,
                                const std::vector<int64_t> &sa, const std::vector<int64_t> &sb, tc_calibration_t *out) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        if (e0) cudaEventDestroy(e0);
        return cuda_fail(cudaErrorMemoryAllocation, "calibrate events");
    }
    tc_status st = TC_OK;
    for (int dir = 0; dir < 2 && st == TC_OK; ++dir) {
        const bool gather = dir == 0;
        cudaStream_t s = gather ? s_off : s_up;
        int64_t best_ok = 0;
        bool still = true;
        for (int64_t m = 1; m <= std::min<int64_t>(k, 64) && st == TC_OK; m *= 2) {
            std::vector<XferDesc> d(gather ? da.begin() : db.begin(), (gather ? da.begin() : db.begin()) + m);
            std::vector<int64_t> sl(gather ? sa.begin() : sb.begin(), (gather ? sa.begin() : sb.begin()) + m);
            double t[2] = {1e30, 1e30};
            for (int rep = 0; rep < 6 && st == TC_OK; ++rep) {
                for (int c = 0; c < 2 && st == TC_OK; ++c) {
                    if (cudaStreamSynchronize(s) != cudaSuccess || cudaEventRecord(e0, s) != cudaSuccess) {
                        st = cuda_fail(cudaGetLastError(), "calibrate small");
                        break;
                    }
                    if ((st = enqueue_xfer(gather, c == 0 ? TC_XFER_DIRECT : TC_XFER_STAGED, d, sl, s)) != TC_OK) break;
                    float ms = 0.f;
                    if (cudaEventRecord(e1, s) != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess ||
                        cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) {
                        st = cuda_fail(cudaGetLastError(), "calibrate small timing");
                        break;
                    }
                    if (rep > 0) t[c] = std::min(t[c], (double)ms);
                }
            }
            if (st != TC_OK) break;
            if (still && t[0] <= t[1]) best_ok = m * B;
            else still = false;
        }
        if (st == TC_OK) {
            auto_direct_bytes[dir] = best_ok;
            out->direct_max_bytes[dir] = best_ok;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return st;
}

tc_status Pool::calibrate(int64_t probe_bytes, tc_calibration_t *out) {
    if (meta_only) return TC_E_NODEV;
    if (cuda_dead) return TC_E_CUDA;
    if (probe_bytes <= 0 || !out) return TC_E_INVAL;
    for (cudaStream_t s : {s_up, s_off, s_up_k, s_off_k}) TC_CUDA(cudaStreamSynchronize(s), "calibrate drain");
    int64_t k = std::max<int64_t>(1, probe_bytes / B);
    k = std::min<int64_t>({k, N / 2, slots.nfree / 2});
    if (k < 1) return TC_E_NOHOST;
    std::vector<XferDesc> da(k), db(k);
    std::vector<int64_t> sa(k), sb(k), sfree(2 * k);
    slots.choose(2 * k, sfree.data());             // free slots, used as scratch while the streams are drained
    for (int64_t i = 0; i < k; ++i) {              // A = blocks [0, k) (read), B = [k, 2k) (rewritten with itself)
        da[i] = XferDesc{(int32_t)i, -1, 0};
        db[i] = XferDesc{(int32_t)(k + i), -1, 0};
        sa[i] = sfree[i];
        sb[i] = sfree[k + i];
    }
    const bool saved_auto[2] = {auto_dir[0], auto_dir[1]};
    auto_dir[0] = auto_dir[1] = false;              // probe sizes exactly as given (no small-batch DIRECT)
    tc_status st = enqueue_xfer(true, TC_XFER_STAGED, db, sb, s_off);   // B's images, so the scatters restore B
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
    double best[4] = {1e30, 1e30, 1e30, 1e30};
    const int32_t modes[2] = {TC_XFER_DIRECT, TC_XFER_STAGED};
    if (st == TC_OK && (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess ||
                        cudaEventCreate(&e2) != cudaSuccess))
        st = cuda_fail(cudaErrorMemoryAllocation, "calibrate events");
    for (int rep = 0; st == TC_OK && rep < 4; ++rep) {
        for (int c = 0; st == TC_OK && c < 4; ++c) {
            if (cudaStreamSynchronize(s_off) != cudaSuccess || cudaStreamSynchronize(s_up) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "calibrate sync");
                break;
            }
            if (cudaEventRecord(e0, s_off) != cudaSuccess || cudaStreamWaitEvent(s_up, e0, 0) != cudaSuccess ||
                cudaStreamWaitEvent(s_up_k, e0, 0) != cudaSuccess || cudaStreamWaitEvent(s_off_k, e0, 0) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "calibrate event");
                break;
            }
            if ((st = enqueue_xfer(true, modes[c >> 1], da, sa, s_off)) != TC_OK) break;
            if ((st = enqueue_xfer(false, modes[c & 1], db, sb, s_up)) != TC_OK) break;
            if (cudaEventRecord(e1, s_off) != cudaSuccess || cudaEventRecord(e2, s_up) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "calibrate event");
                break;
            }
            float t1 = 0.f, t2 = 0.f;
            if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventSynchronize(e2) != cudaSuccess ||
                cudaEventElapsedTime(&t1, e0, e1) != cudaSuccess || cudaEventElapsedTime(&t2, e0, e2) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "calibrate timing");
                break;
            }
            if (rep > 0) best[c] = std::min(best[c], (double)std::max(t1, t2));   // rep 0 warms every path up
        }
    }
    for (cudaEvent_t e : {e0, e1, e2})
        if (e) cudaEventDestroy(e);
    if (st == TC_OK) st = calibrate_small(k, da, db, sa, sb, out);
    auto_dir[0] = saved_auto[0];
    auto_dir[1] = saved_auto[1];
    if (st != TC_OK) return st;
    int bc = 3;
    for (int c = 0; c < 4; ++c)
        if (best[c] < best[bc]) bc = c;
    auto_choice[0] = modes[bc >> 1];
    auto_choice[1] = modes[bc & 1];
    if (auto_dir[0]) mode_d2h = auto_choice[0];
    if (auto_dir[1]) mode_h2d = auto_choice[1];
    out->d2h = auto_choice[0];
    out->h2d = auto_choice[1];
    out->probe_bytes = k * B;
    for (int c = 0; c < 4; ++c) out->gbs[c] = 2.0 * (double)(k * B) / (best[c] * 1e-3) / 1e9;
    return TC_OK;
}

// COPY mode: one strided 2-D DMA per block (2L rows of C bytes; pool row pitch N*C, slot rows packed); the table
// epilogue is a small kernel in stream order (offload: first, upload: after the data has landed).
tc_status Pool::xfer_copy2d(XferJob &j) {
    const auto &slot_of = *j.slot_of;
    cudaEvent_t t0;
    tc_status st;
    const int64_t table_launches = (j.n + kMaxInlineDesc - 1) / kMaxInlineDesc;
    if (j.gather) {
        TC_CUDA(launch_table(true, j.desc->data(), j.n, table_dev, j.s), "table kernel");
        n_launch += table_launches;
    }
    if ((st = span_begin(j.s, &t0, /*kernel=*/false)) != TC_OK) return st;
    for (int64_t i = 0; i < j.n; ++i) {
        char *pool_p = kv + (int64_t)(*j.desc)[i].blk * C;
        char *host_p = host_ptr(slot_of[i]);
        if (j.gather)
            TC_CUDA(cudaMemcpy2DAsync(host_p, (size_t)C, pool_p, (size_t)(N * C), (size_t)C, (size_t)(2 * L),
                                      cudaMemcpyDeviceToHost, j.s), "2D memcpy");
        else
            TC_CUDA(cudaMemcpy2DAsync(pool_p, (size_t)(N * C), host_p, (size_t)C, (size_t)C, (size_t)(2 * L),
                                      cudaMemcpyHostToDevice, j.s), "2D memcpy");
        ++n_memcpy;
    }
    trace(j.gather ? "d2h" : "h2d");
    if ((st = span_end(j.s, j.gather ? 3 : 4, t0, j.n * B)) != TC_OK) return st;
    if (!j.gather) {
        TC_CUDA(launch_table(false, j.desc->data(), j.n, table_dev, j.s), "table kernel");
        n_launch += table_launches;
    }
    return TC_OK;
}

// Staging address of piece p: contiguous by block index, or one of two halves when double-buffering.
char *Pool::xfer_base(const XferJob &j, int64_t p) const {
    if (!j.ring_reuse) return j.stg + j.cut[p] * B;
    return j.stg + (p % 2) * j.pb * B;                 // pieces alternate the two halves (each <= pb blocks)
}

tc_status Pool::ev_rec(cudaStream_t st, int32_t *out) {
    *out = event_get();
    if (*out < 0) return cuda_fail(cudaErrorMemoryAllocation, "event pool");
    TC_CUDA(cudaEventRecord(events[*out], st), "piece event");
    return TC_OK;
}

// Copy-engine DMA of pieces [a, b) between the staging slot `base` and the host slots: one cudaMemcpyAsync per
// contiguous run of host slots (one run for a batch whose slots HostSlots::choose found contiguous).
tc_status Pool::xfer_copy(XferJob &j, int64_t a, int64_t b, char *base) {
    const bool to_host = j.gather;
    const auto &slot_of = *j.slot_of;
    cudaEvent_t t0;
    tc_status s0 = span_begin(j.s, &t0, /*kernel=*/false);
    if (s0 != TC_OK) return s0;
    cp_dst.clear(); cp_src.clear(); cp_size.clear();
    for (int64_t i = a; i < b;) {
        int64_t k = i + 1;
        char *hp = host_ptr(slot_of[i]);
        while (k < b && host_ptr(slot_of[k]) == hp + (k - i) * B) ++k;   // contiguous run of host memory
        char *dp = base + (i - a) * B;
        cp_dst.push_back(to_host ? (void *)hp : (void *)dp);
        cp_src.push_back(to_host ? (void *)dp : (void *)hp);
        cp_size.push_back((size_t)((k - i) * B));
        i = k;
    }
    for (size_t r = 0; r < cp_dst.size(); ++r) {
        TC_CUDA(cudaMemcpyAsync(cp_dst[r], cp_src[r], cp_size[r],
                                to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, j.s),
                "staged memcpy");
        ++n_memcpy;
    }
    trace(to_host ? "d2h" : "h2d");
    return span_end(j.s, to_host ? 3 : 4, t0, (b - a) * B);
}

// Launches the gather/scatter of n descriptors (by value in the kernel parameters, at most kMaxInlineDesc per
// launch) with path's launch configuration; `kind` names the timing slot (0 offload, 1 upload, 2 device tier).
tc_status Pool::launch_descs(bool gather, int32_t kind, int path, const XferDesc *d, int64_t n, cudaStream_t s) {
    if (check) check_descs(kind, d, n);
    for (int64_t a = 0; a < n; a += kMaxInlineDesc) {
        const int32_t m = (int32_t)std::min<int64_t>(kMaxInlineDesc, n - a);
        const XferGeom g = geom(kind, m * B);
        TC_CUDA(launch_xfer(gather, d + a, m, g, kv, table_dev, ctas[path], nthreads[path], variant[path], s),
                gather ? "gather kernel" : "scatter kernel");
        trace(gather ? "gather" : "scatter");
        ++n_launch;
    }
    return TC_OK;
}

// Device-side gather/scatter of pieces [a, b) against the staging slot `base`.
tc_status Pool::xfer_kernel(XferJob &j, int64_t a, int64_t b, char *base) {
    cd_.resize((size_t)(b - a));
    for (int64_t i = a; i < b; ++i) {
        cd_[i - a] = (*j.desc)[i];
        cd_[i - a].ext = reinterpret_cast<uint64_t>(base + (i - a) * B);
    }
    cudaEvent_t t0;
    tc_status st = span_begin(j.sk, &t0);
    if (st != TC_OK) return st;
    if ((st = launch_descs(j.gather, j.gather ? 0 : 1, 2, cd_.data(), b - a, j.sk)) != TC_OK) return st;
    return span_end(j.sk, j.gather ? 0 : 1, t0, (b - a) * B, /*link=*/false);
}

tc_status Pool::xfer_phase_a(XferJob &j) {
    if (j.n == 0) return TC_OK;
    tc_status st;
    if (j.mode == TC_XFER_COPY) return xfer_copy2d(j);
    if (j.mode == TC_XFER_DIRECT) {
        const bool dev_tier = j.slot_of == nullptr || j.slot_of->empty();
        const int path = dev_tier ? 2 : (j.gather ? 0 : 1);
        const int32_t kind = dev_tier ? 2 : (j.gather ? 7 : 8);
        const XferDesc *d = j.desc->data();
        if (!dev_tier) {
            cd_.resize((size_t)j.n);
            for (int64_t i = 0; i < j.n; ++i) {
                cd_[i] = (*j.desc)[i];
                cd_[i].ext = reinterpret_cast<uint64_t>(host_dev_ptr((*j.slot_of)[i]));
            }
            d = cd_.data();
        }
        cudaEvent_t t0;
        if ((st = span_begin(j.s, &t0)) != TC_OK) return st;
        if ((st = launch_descs(j.gather, kind, path, d, j.n, j.s)) != TC_OK) return st;
        return span_end(j.s, kind, t0, j.n * B);
    }
    if (j.need_hop) {                                // the aux stream starts after the main stream's waits
        int32_t e0;
        if ((st = ev_rec(j.s, &e0)) != TC_OK) return st;
        TC_CUDA(cudaStreamWaitEvent(j.sk, events[e0], 0), "aux wait");
    }
    std::vector<int32_t> done(j.ring_reuse ? j.npieces : 0, -1);
    for (int64_t p = 0; p < j.npieces; ++p) {
        const int64_t a = j.cut[p], b = j.cut[p + 1];
        char *base = xfer_base(j, p);
        if (j.gather) {
            if (j.ring_reuse && p >= 2) TC_CUDA(cudaStreamWaitEvent(j.sk, events[done[p - 2]], 0), "ring reuse");
            if ((st = piece_waits(j, a, b, j.sk)) != TC_OK) return st;       // the gather reads the items' blocks
            if ((st = xfer_kernel(j, a, b, base)) != TC_OK) return st;
            // the D2H copy of a piece is issued right after its gather, so the link starts after the small
            // head piece's gather and a handful of API calls
            if (j.sk != j.s) {
                if ((st = ev_rec(j.sk, &j.ev[p])) != TC_OK) return st;
                TC_CUDA(cudaStreamWaitEvent(j.s, events[j.ev[p]], 0), "gather->D2H wait");
            }
            if ((st = xfer_copy(j, a, b, base)) != TC_OK) return st;
            if (j.ring_reuse && (st = ev_rec(j.s, &done[p])) != TC_OK) return st;
            if (j.item_dep) {                            // piece p is on the host
                if (j.ring_reuse) j.piece_done[p] = done[p];
                else if ((st = ev_rec(j.s, &j.piece_done[p])) != TC_OK) return st;
            }
        } else {
            if (j.ring_reuse && p >= 2) TC_CUDA(cudaStreamWaitEvent(j.s, events[done[p - 2]], 0), "ring reuse");
            if ((st = piece_waits(j, a, b, j.s)) != TC_OK) return st;        // the H2D reads the items' host slots
            if ((st = xfer_copy(j, a, b, base)) != TC_OK) return st;
            if (j.sk != j.s && (st = ev_rec(j.s, &j.ev[p])) != TC_OK) return st;
            if (j.ring_reuse) {
                TC_CUDA(cudaStreamWaitEvent(j.sk, events[j.ev[p]], 0), "H2D->scatter wait");
                if ((st = xfer_kernel(j, a, b, base)) != TC_OK) return st;
                if ((st = ev_rec(j.sk, &done[p])) != TC_OK) return st;
                if (j.item_dep) j.piece_done[p] = done[p];   // piece p is in the pool, its table entries remapped
            }
        }
    }
    if (j.ring_reuse && !j.gather) TC_CUDA(cudaStreamWaitEvent(j.s, events[done[j.npieces - 1]], 0), "join");
    return TC_OK;
}

tc_status Pool::xfer_phase_b(XferJob &j) {
    if (j.n == 0 || j.mode != TC_XFER_STAGED) return TC_OK;
    tc_status st;
    if (!j.ring_reuse && !j.gather) {
        for (int64_t p = 0; p < j.npieces; ++p) {
            const int64_t a = j.cut[p], b = j.cut[p + 1];
            if (j.sk != j.s) TC_CUDA(cudaStreamWaitEvent(j.sk, events[j.ev[p]], 0), "H2D->scatter wait");
            if ((st = xfer_kernel(j, a, b, xfer_base(j, p))) != TC_OK) return st;
            if (j.item_dep && (st = ev_rec(j.sk, &j.piece_done[p])) != TC_OK) return st;
        }
        if (j.half < 0 && j.sk != j.s) {              // the upload completes when its last scatter has
            int32_t last;
            if ((st = ev_rec(j.sk, &last)) != TC_OK) return st;
            TC_CUDA(cudaStreamWaitEvent(j.s, events[last], 0), "scatter->upload join");
        }
    }
    // staging fences for the halves mode: the stream on which this batch's last staging access completes (gather:
    // the D2H on the main stream; halves upload: the scatter on the main stream; other uploads: joined into j.s)
    const int dir = j.gather ? 0 : 1;
    if (j.half >= 0) {
        TC_CUDA(cudaEventRecord(half_free[dir][j.half], j.gather ? j.s : j.sk), "half free");
    } else {                                           // a whole-buffer batch: both halves were (maybe) touched
        TC_CUDA(cudaEventRecord(half_free[dir][0], j.s), "half free");
        TC_CUDA(cudaEventRecord(half_free[dir][1], j.s), "half free");
    }
    return TC_OK;
}

tc_status Pool::enqueue_xfer(bool gather, int32_t mode, const std::vector<XferDesc> &desc,
                             const std::vector<int64_t> &slot_of, cudaStream_t s) {
    XferJob j;
    tc_status st = xfer_init(j, gather, mode, &desc, &slot_of, s);
    if (st == TC_OK) st = xfer_phase_a(j);
    if (st == TC_OK) st = xfer_phase_b(j);
    return st;
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
    // Without a compute stream the push runs on s_off, and a later offload's gather may run on the aux stream
    // s_off_k (staging halves), which is not ordered after s_off: its table epilogue (-1) must not be overwritten
    // by this push landing late.  offload_waits makes s_off_k wait on this event.
    if (!s_compute) {
        if (!ag.push_ev) TC_CUDA(cudaEventCreateWithFlags(&ag.push_ev, cudaEventDisableTiming), "push event");
        TC_CUDA(cudaEventRecord(ag.push_ev, s), "push event");
    }
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
    ag.table.reserve((size_t)(pos0 + k));             // the only allocation; before any state changes
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

// a2 admission: validate everything before touching state (A5, A15), item by item in order so that the first failing
// item decides the status (sequential-composition semantics of a batch, reading B1).
tc_status Pool::plan_offload(OffPlan &P, int32_t na, const int32_t *ags, const int64_t *off, const int32_t *ids) {
    if (na < 1 || !ags || !off || !ids || off[0] != 0) return TC_E_INVAL;
    if (++epoch == 0) { std::fill(stamp.begin(), stamp.end(), 0); epoch = 1; }
    // per item, in order (B1: the first failing item's status): validity, then the tier — the whole offload to the
    // peer tier if its free list holds it, else to the CPU block buffer, else refused (reading C1)
    const int64_t hf = slots.nfree, pf = (int64_t)peer.free_list.size();
    int64_t ht = 0, pt = 0;
    std::vector<uint8_t> to_peer(na, 0);
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
        if (unbuffered) continue;
        const int64_t m = off[k + 1] - off[k];
        if (pf - pt >= m) {
            to_peer[k] = 1;
            pt += m;
        } else if (hf - ht >= m) {
            ht += m;
        } else {
            return TC_E_NOHOST;
        }
    }
    P.na = na; P.ags = ags; P.off = off; P.ids = ids;
    const int64_t n = off[na];
    P.desc.resize(n);
    P.slot_of.resize(n);
    P.host_taken = P.peer_taken = 0;
    if (!unbuffered) {       // peer tier: LIFO pops (A16); host tier: one contiguous run for the batch (A16')
        P.host_slots.resize(ht);
        slots.choose(ht, P.host_slots.data());
        for (int32_t k = 0; k < na; ++k)
            for (int64_t i = off[k]; i < off[k + 1]; ++i)
                P.slot_of[i] = to_peer[k] ? peer.free_list[pf - 1 - P.peer_taken++] : P.host_slots[P.host_taken++];
    }
    if (unbuffered) {
        // Fig. 11 ablation: no CPU block buffer — pinned host memory is allocated for this offload now and freed
        // when its upload retires (the bursty OS allocation pattern of P:470-479).
        char *h = nullptr;
        if (meta_only) {
            h = nullptr;
        } else if (cudaHostAlloc(reinterpret_cast<void **>(&h), (size_t)(n * B),
                                 cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return TC_E_NOHOST;
        }
        char *dh = nullptr;
        if (h) cudaHostGetDevicePointer(reinterpret_cast<void **>(&dh), h, 0);
        extra[next_slot] = ExtraSlab{h, dh, n, n};
        for (int64_t i = 0; i < n; ++i) P.slot_of[i] = next_slot + i;
        next_slot += n;
    }
    for (int32_t k = 0; k < na; ++k)
        for (int64_t i = off[k]; i < off[k + 1]; ++i)
            P.desc[i] = XferDesc{ids[i], ags[k] * max_bpa + alloc.own_pos[ids[i]], 0};
    split_tiers(P.desc, P.slot_of, P.ts);
    // everything commit_offload stores is built (and its containers grown) here, before any state changes: a
    // std::bad_alloc leaves the pool untouched (TC_E_OOM), and the commit itself cannot fail
    P.pend.assign(na, {});
    P.newh.clear();
    P.newh.reserve(na);
    for (int32_t k = 0; k < na; ++k) {
        HandleRec hr;
        hr.agent = ags[k];
        hr.cls = agents[ags[k]].cls;
        hr.state = kOffloaded;
        const int64_t m = off[k + 1] - off[k];
        hr.pos.reserve(m);
        hr.slots.reserve(m);
        P.pend[k].reserve(m);
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            hr.pos.push_back(alloc.own_pos[ids[i]]);
            hr.slots.push_back(P.slot_of[i]);
            P.pend[k].push_back(ids[i]);
        }
        P.newh.emplace(next_handle + (tc_handle)k, std::move(hr));
    }
    pending_dev.reserve(pending_dev.size() + na);
    pending_epoch.reserve(pending_epoch.size() + na);
    handles.reserve(handles.size() + na);
    return TC_OK;
}

// Host-tier blocks keep their slot ids (the transfer engine resolves them); peer-tier blocks get ext = the peer slot.
void Pool::split_tiers(const std::vector<XferDesc> &desc, const std::vector<int64_t> &slot_of, TierSplit &ts) const {
    ts.hdesc.clear();
    ts.hslot.clear();
    ts.pdesc.clear();
    if (peer.count == 0) return;                    // no peer tier: the plan's own vectors are used as they are
    for (size_t i = 0; i < desc.size(); ++i) {
        if (is_peer(slot_of[i])) {
            XferDesc d = desc[i];
            d.ext = reinterpret_cast<uint64_t>(peer_ptr(slot_of[i]));
            ts.pdesc.push_back(d);
        } else {
            ts.hdesc.push_back(desc[i]);
            ts.hslot.push_back(slot_of[i]);
        }
    }
}

// The peer-tier part of a batch: one device-side kernel on the direction's aux stream, started after the main
// stream's waits; *join_ev = its completion (the main stream joins it after enqueueing the host-tier part).
tc_status Pool::peer_launch(bool gather, const std::vector<XferDesc> &pd, cudaStream_t s, int32_t *join_ev) {
    *join_ev = -1;
    if (pd.empty() || meta_only) return TC_OK;
    cudaStream_t aux = gather ? s_off_k : s_up_k;
    int32_t e0;
    tc_status st = ev_rec(s, &e0);
    if (st != TC_OK) return st;
    TC_CUDA(cudaStreamWaitEvent(aux, events[e0], 0), "peer wait");
    const int32_t kind = gather ? 5 : 6;
    cudaEvent_t t0;
    if ((st = span_begin(aux, &t0)) != TC_OK) return st;
    if ((st = launch_descs(gather, kind, 3, pd.data(), (int64_t)pd.size(), aux)) != TC_OK) return st;
    if ((st = span_end(aux, kind, t0, (int64_t)pd.size() * B, /*link=*/false)) != TC_OK) return st;
    return ev_rec(aux, join_ev);
}

tc_status Pool::join(cudaStream_t s, int32_t ev) {
    if (ev >= 0) TC_CUDA(cudaStreamWaitEvent(s, events[ev], 0), "peer join");
    return TC_OK;
}

// GPU-side dependencies of an offload: the compute stream (the agents' last decode writes) and any upload into
// these agents since the last sync.
tc_status Pool::offload_waits(const OffPlan &P, bool ups) {
    if (s_compute) {
        TC_CUDA(cudaEventRecord(ev_compute, s_compute), "compute event");
        TC_CUDA(cudaStreamWaitEvent(s_off, ev_compute, 0), "compute wait");
    }
    if (s_compute) TC_CUDA(cudaStreamWaitEvent(s_off_k, ev_compute, 0), "compute wait");
    for (int32_t k = 0; k < P.na; ++k) {
        if (cudaEvent_t pe = agents[P.ags[k]].push_ev)
            TC_CUDA(cudaStreamWaitEvent(s_off_k, pe, 0), "table push->offload wait");
        const int32_t ue = ups ? agents[P.ags[k]].up_event : -1;
        if (ue >= 0) {
            TC_CUDA(cudaStreamWaitEvent(s_off, events[ue], 0), "upload->offload wait");
            TC_CUDA(cudaStreamWaitEvent(s_off_k, events[ue], 0), "upload->offload wait");   // halves gathers
        }
    }
    return TC_OK;
}

// commit (a3 logical effects + a4 pending free); ev = the offload's completion event
// (no allocation: plan_offload built the handle records and grew every container this touches)
void Pool::commit_offload(OffPlan &P, int32_t ev, tc_handle *out, const std::vector<int32_t> *item_ev) {
    const int64_t n = P.off[P.na];
    if (!unbuffered) {
        slots.take(P.host_slots.data(), P.host_taken);
        peer.free_list.resize(peer.free_list.size() - P.peer_taken);
    }
    for (int32_t k = 0; k < P.na; ++k) {
        const int32_t a = P.ags[k];
        AgentRec &ag = agents[a];
        for (int64_t i = P.off[k]; i < P.off[k + 1]; ++i) {
            const int32_t b = P.ids[i];
            ag.table[alloc.own_pos[b]] = -1;               // location flag -> host
            alloc.state[b] = kPending;                     // pending free until tc_sync
            alloc.own_agent[b] = -1;
            alloc.own_pos[b] = -1;
        }
        pending_dev.emplace_back(ag.cls, std::move(P.pend[k]));
        pending_epoch.push_back(epoch_id);
        ++ag.live_offloads;
        const tc_handle h = next_handle++;
        P.newh.at(h).ev = item_ev ? (*item_ev)[k] : ev;
        out[k] = h;
    }
    handles.merge(P.newh);                                 // splices the prebuilt nodes (no rehash: reserved)
    if (!meta_only) bytes_d2h += n * B;
}

// validate + a5 dry run on counters only, item by item in order.  Blocks already claimed by a gradual reservation
// are used first (claim order); only the remainder is allocated, lowest free first.
tc_status Pool::plan_upload(UpPlan &P, int32_t nh, const tc_handle *hs, const int64_t *off) {
    if (nh < 1 || !hs || !off || off[0] != 0) return TC_E_INVAL;
    P.hr.assign(nh, nullptr);
    P.rr.assign(nh, 0);
    P.need.assign(nh, 0);
    std::vector<int64_t> cl = alloc.claimed;
    int64_t nf = alloc.nfree;
    std::unordered_set<tc_handle> seen;
    for (int32_t k = 0; k < nh; ++k) {
        auto it = handles.find(hs[k]);
        if (it == handles.end() || it->second.state != kOffloaded || !seen.insert(hs[k]).second) return TC_E_HANDLE;
        P.hr[k] = &it->second;
        const int64_t k_n = off[k + 1] - off[k];
        if (k_n != (int64_t)P.hr[k]->pos.size()) return TC_E_INVAL;
        P.need[k] = k_n - (int64_t)P.hr[k]->resv.size();
        const int64_t r = P.need[k] > 0 ? BlockAllocator::plan(P.hr[k]->cls, P.need[k], nf, alloc.reserved, cl) : 0;
        if (r < 0) return TC_E_NOBLOCKS;      // upload "stalls"; handles stay valid
        P.rr[k] = r;
        cl[P.hr[k]->cls] += r;
        nf -= std::max<int64_t>(0, P.need[k]);
    }
    P.nh = nh; P.hs = hs; P.off = off;
    const int64_t n = off[nh];
    P.n_fresh = 0;
    for (int32_t k = 0; k < nh; ++k) P.n_fresh += P.need[k];
    // sequential composition of lowest-free-first == the n_fresh lowest free ids split in order
    std::vector<int32_t> fresh(P.n_fresh);
    {
        int64_t got = 0;
        for (int64_t w = alloc.hint; got < P.n_fresh && w < (int64_t)alloc.bits.size(); ++w)
            for (uint64_t x = alloc.bits[w]; x && got < P.n_fresh; x &= x - 1)
                fresh[got++] = (int32_t)(w * 64 + __builtin_ctzll(x));
    }
    P.dst.resize(n);
    P.desc.resize(n);
    P.slot_of.resize(n);
    int64_t f = 0;
    for (int32_t k = 0; k < nh; ++k) {
        int64_t i = off[k];
        for (int32_t b : P.hr[k]->resv) P.dst[i++] = b;
        for (; i < off[k + 1]; ++i) P.dst[i] = fresh[f++];
        for (i = off[k]; i < off[k + 1]; ++i) {
            const int64_t q = i - off[k];
            P.desc[i] = XferDesc{P.dst[i], P.hr[k]->agent * max_bpa + P.hr[k]->pos[q], 0};
            P.slot_of[i] = P.hr[k]->slots[q];
        }
    }
    split_tiers(P.desc, P.slot_of, P.ts);
    P.taken.resize(P.n_fresh);                    // commit_upload allocates nothing (strong guarantee on OOM)
    slots.released.reserve(slots.released.size() + n);
    slots.released_epoch.reserve(slots.released_epoch.size() + n);
    return TC_OK;
}

tc_status Pool::upload_waits(const UpPlan &P) {          // A13: the upload waits for each handle's offload
    for (int32_t k = 0; k < P.nh; ++k)
        if (P.hr[k]->ev >= 0) {
            TC_CUDA(cudaStreamWaitEvent(s_up, events[P.hr[k]->ev], 0), "offload->upload wait");
            TC_CUDA(cudaStreamWaitEvent(s_up_k, events[P.hr[k]->ev], 0), "offload->upload wait");   // halves H2D
        }
    return TC_OK;
}

// commit (a5 allocation, a6 remap, a7 released slots); ev = the upload's completion event
void Pool::commit_upload(UpPlan &P, int32_t ev, int32_t *out_ids, const std::vector<int32_t> *item_ev) {
    if (P.n_fresh > 0) alloc.take_lowest(P.n_fresh, P.taken.data());   // == the planned ids (nothing changed since)
    for (int32_t k = 0; k < P.nh; ++k) {
        HandleRec &h = *P.hr[k];
        AgentRec &ag = agents[h.agent];
        alloc.claimed[h.cls] += P.rr[k];
        n_reserved -= (int64_t)h.resv.size();
        for (int64_t i = P.off[k]; i < P.off[k + 1]; ++i) {
            const int64_t q = i - P.off[k];
            const int32_t b = P.dst[i];
            alloc.state[b] = kAlloc;
            alloc.own_agent[b] = h.agent;
            alloc.own_pos[b] = h.pos[q];
            ag.table[h.pos[q]] = b;                        // fused remap's host mirror (A6)
            slots.released.push_back(h.slots[q]);
            slots.released_epoch.push_back(epoch_id);
            out_ids[i] = b;
        }
        h.resv.clear();
        h.plan.clear();
        resv_active.erase(P.hs[k]);
        h.state = kUploaded;
        h.up_epoch = epoch_id;
        h.ev = item_ev ? (*item_ev)[k] : ev;
        --ag.live_offloads;
        ag.up_event = h.ev;
    }
    if (!meta_only) bytes_h2d += P.off[P.nh] * B;
}

tc_status Pool::offload_batch(int32_t na, const int32_t *ags, const int64_t *off, const int32_t *ids,
                              tc_handle *out) {
    if (cuda_dead) return TC_E_CUDA;
    if (trace_cap > 0) trace_t0 = steady_ns();
    if (!out) return TC_E_INVAL;
    OffPlan P;
    tc_status st = plan_offload(P, na, ags, off, ids);
    if (st != TC_OK) return st;
    int32_t ev = -1;
    std::vector<int32_t> deps, item_ev;
    bool fine = false;
    if (!meta_only) try {
        XferJob j;
        const bool pt = peer.count > 0;
        if ((st = xfer_init(j, true, mode_d2h, pt ? &P.ts.hdesc : &P.desc, pt ? &P.ts.hslot : &P.slot_of, s_off,
                            pt ? nullptr : off, na)) != TC_OK)
            return st;
        if (!pt) {
            deps.resize(na);
            for (int32_t k = 0; k < na; ++k) deps[k] = agents[ags[k]].up_event;
            fine = fine_grained(j, off, na, deps);
        }
        if ((st = offload_waits(P, !fine)) != TC_OK) return st;
        int32_t pj;
        if ((st = peer_launch(true, P.ts.pdesc, s_off, &pj)) != TC_OK) return st;
        if ((st = xfer_phase_a(j)) != TC_OK) return st;
        if ((st = xfer_phase_b(j)) != TC_OK) return st;
        if ((st = join(s_off, pj)) != TC_OK) return st;
        if ((st = ev_rec(s_off, &ev)) != TC_OK) return st;
        if (fine) item_events(j, item_ev);
    } catch (const std::bad_alloc &) {
        return enqueue_oom();
    }
    commit_offload(P, ev, out, fine ? &item_ev : nullptr);
    trace_calls(1, ags, out, off, na, s_off);
    return TC_OK;
}

tc_status Pool::upload_batch(int32_t nh, const tc_handle *hs, const int64_t *off, int32_t *out_ids) {
    if (cuda_dead) return TC_E_CUDA;
    if (trace_cap > 0) trace_t0 = steady_ns();
    if (!out_ids) return TC_E_INVAL;
    UpPlan P;
    tc_status st = plan_upload(P, nh, hs, off);
    if (st != TC_OK) return st;
    int32_t ev = -1;
    std::vector<int32_t> deps, item_ev;
    bool fine = false;
    if (!meta_only) try {
        XferJob j;
        const bool pt = peer.count > 0;
        if ((st = xfer_init(j, false, mode_h2d, pt ? &P.ts.hdesc : &P.desc, pt ? &P.ts.hslot : &P.slot_of, s_up,
                            pt ? nullptr : off, nh)) != TC_OK)
            return st;
        if (!pt) {
            deps.resize(nh);
            for (int32_t k = 0; k < nh; ++k) deps[k] = P.hr[k]->ev;
            fine = fine_grained(j, off, nh, deps);
        }
        if (!fine && (st = upload_waits(P)) != TC_OK) return st;
        int32_t pj;
        if ((st = peer_launch(false, P.ts.pdesc, s_up, &pj)) != TC_OK) return st;
        if ((st = xfer_phase_a(j)) != TC_OK) return st;
        if ((st = xfer_phase_b(j)) != TC_OK) return st;
        if ((st = join(s_up, pj)) != TC_OK) return st;
        if ((st = ev_rec(s_up, &ev)) != TC_OK) return st;
        if (fine) item_events(j, item_ev);
    } catch (const std::bad_alloc &) {
        return enqueue_oom();
    }
    commit_upload(P, ev, out_ids, fine ? &item_ev : nullptr);
    trace_calls(2, nullptr, hs, off, nh, s_up);
    return TC_OK;
}

// a8: one scheduling cycle = this cycle's uploads, then its offloads, as one call.  Both are validated
// before anything changes (all-or-nothing; uploads' status first).  The offloads are validated against the pre-cycle
// state, so they cannot name blocks this cycle's uploads allocate (reading B5).  The two directions are enqueued
// interleaved — H2D copies, gathers, D2H copies, scatters — so both links start as early as possible.
tc_status Pool::cycle(int32_t nh, const tc_handle *hs, const int64_t *up_off, int32_t *out_ids, int32_t na,
                      const int32_t *ags, const int64_t *off_off, const int32_t *ids, tc_handle *out_h) {
    if (cuda_dead) return TC_E_CUDA;
    if (nh < 0 || na < 0 || (nh > 0 && !out_ids) || (na > 0 && !out_h)) return TC_E_INVAL;
    if (trace_cap > 0) trace_t0 = steady_ns();
    if (g_trace) {
        g_trace_t0 = std::chrono::steady_clock::now();
        g_trace_buf = "[tc trace] cycle";
    }
    UpPlan U;
    OffPlan O;
    tc_status st;
    if (nh > 0 && (st = plan_upload(U, nh, hs, up_off)) != TC_OK) return st;
    if (na > 0 && (st = plan_offload(O, na, ags, off_off, ids)) != TC_OK) return st;
    trace("plans");
    int32_t ev_up = -1, ev_off = -1;
    std::vector<int32_t> deps_u, deps_o, iev_u, iev_o;
    bool fine_u = false, fine_o = false;
    if (!meta_only) try {
        XferJob ju, jo;
        int32_t pu = -1, po = -1;                                     // peer-tier parts (NEXT-2)
        const bool pt = peer.count > 0;
        if (nh > 0) {
            if ((st = xfer_init(ju, false, mode_h2d, pt ? &U.ts.hdesc : &U.desc, pt ? &U.ts.hslot : &U.slot_of,
                                s_up, pt ? nullptr : up_off, nh)) != TC_OK)
                return st;
            if (!pt) {
                deps_u.resize(nh);
                for (int32_t k = 0; k < nh; ++k) deps_u[k] = U.hr[k]->ev;
                fine_u = fine_grained(ju, up_off, nh, deps_u);
            }
            if (!fine_u && (st = upload_waits(U)) != TC_OK) return st;
            if ((st = peer_launch(false, U.ts.pdesc, s_up, &pu)) != TC_OK) return st;
            if ((st = xfer_phase_a(ju)) != TC_OK) return st;          // H2D copies start first
        }
        if (na > 0) {
            if ((st = xfer_init(jo, true, mode_d2h, pt ? &O.ts.hdesc : &O.desc, pt ? &O.ts.hslot : &O.slot_of,
                                s_off, pt ? nullptr : off_off, na)) != TC_OK)
                return st;
            if (!pt) {
                deps_o.resize(na);
                for (int32_t k = 0; k < na; ++k) deps_o[k] = agents[ags[k]].up_event;
                fine_o = fine_grained(jo, off_off, na, deps_o);
            }
            if ((st = offload_waits(O, !fine_o)) != TC_OK) return st;
            if ((st = peer_launch(true, O.ts.pdesc, s_off, &po)) != TC_OK) return st;
            if ((st = xfer_phase_a(jo)) != TC_OK) return st;          // gathers
            if ((st = xfer_phase_b(jo)) != TC_OK) return st;          // D2H copies
            if ((st = join(s_off, po)) != TC_OK) return st;
            if ((st = ev_rec(s_off, &ev_off)) != TC_OK) return st;
            if (fine_o) item_events(jo, iev_o);
        }
        if (nh > 0) {
            if ((st = xfer_phase_b(ju)) != TC_OK) return st;          // scatters + remap
            if ((st = join(s_up, pu)) != TC_OK) return st;
            if ((st = ev_rec(s_up, &ev_up)) != TC_OK) return st;
            if (fine_u) item_events(ju, iev_u);
        }
    } catch (const std::bad_alloc &) {
        return enqueue_oom();
    }
    if (nh > 0) commit_upload(U, ev_up, out_ids, fine_u ? &iev_u : nullptr);
    if (na > 0) commit_offload(O, ev_off, out_h, fine_o ? &iev_o : nullptr);
    if (nh > 0) trace_calls(2, nullptr, hs, up_off, nh, s_up);
    if (na > 0) trace_calls(1, ags, out_h, off_off, na, s_off);
    if (g_trace) {
        trace("commit");
        std::fprintf(stderr, "%s\n", g_trace_buf.c_str());
    }
    return TC_OK;
}

// ------------------------------------------------------------------------------------------------ NEXT-1
// Gradual GPU Block Reservation: claim an offloaded handle's destination blocks over several
// scheduling ticks so the predictive upload never stalls on allocation.  Chunks are near-equal, largest first;
// each tick claims up to the cumulative target, a shortfall carries to the next tick.
tc_status Pool::reserve_begin(tc_handle h, int32_t cycles) {
    auto it = handles.find(h);
    if (it == handles.end() || it->second.state != kOffloaded) return TC_E_HANDLE;
    HandleRec &hd = it->second;
    if (cycles < 1 || !hd.plan.empty() || !hd.resv.empty()) return TC_E_INVAL;
    const int64_t n = (int64_t)hd.pos.size();
    hd.plan.resize(cycles);
    for (int32_t i = 0; i < cycles; ++i) hd.plan[i] = n / cycles + (i < n % cycles ? 1 : 0);
    hd.ticks = 0;
    resv_active.insert(h);
    return TC_OK;
}

tc_status Pool::reserve_tick() {
    for (tc_handle h : resv_active) {           // issue order (std::set)
        HandleRec &hd = handles[h];
        hd.ticks += 1;
        int64_t target = 0;
        for (int32_t i = 0; i < hd.ticks && i < (int32_t)hd.plan.size(); ++i) target += hd.plan[i];
        const int64_t want = target - (int64_t)hd.resv.size();
        const int64_t uc = alloc.unclaimed(hd.cls);
        const int64_t headroom = std::max<int64_t>(0, alloc.nfree - alloc.unclaimed_sum());
        const int64_t k = std::min({want, alloc.nfree, uc + headroom});
        if (k <= 0) continue;
        const int64_t r = BlockAllocator::plan(hd.cls, k, alloc.nfree, alloc.reserved, alloc.claimed);
        if (r < 0) continue;                     // cannot happen: k <= the largest admissible request
        std::vector<int32_t> ids(k);
        alloc.take_lowest(k, ids.data());
        alloc.claimed[hd.cls] += r;
        for (int32_t b : ids) {
            alloc.state[b] = kReserved;
            hd.resv.push_back(b);
        }
        n_reserved += k;
    }
    return TC_OK;
}

tc_status Pool::reserve_cancel(tc_handle h) {
    auto it = handles.find(h);
    if (it == handles.end() || it->second.state != kOffloaded) return TC_E_HANDLE;
    HandleRec &hd = it->second;
    for (int32_t b : hd.resv) {
        alloc.state[b] = kFree;
        alloc.set_free(b);
    }
    const int64_t k = (int64_t)hd.resv.size();
    alloc.claimed[hd.cls] -= std::min(k, alloc.claimed[hd.cls]);
    n_reserved -= k;
    hd.resv.clear();
    hd.plan.clear();
    hd.ticks = 0;
    resv_active.erase(h);
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
        TC_CUDA(cudaStreamSynchronize(s_up_k), "sync upload aux stream");
        TC_CUDA(cudaStreamSynchronize(s_off_k), "sync offload aux stream");
        if (tc_status st = drain_foreign(); st != TC_OK) return st;
        spans_collect();
        if ((int64_t)kts_meta.size() > kKts / 2) stamps_collect();
        ++sync_count;
    }
    retire_before(epoch_id + 1);          // everything: the streams are drained
    return TC_OK;
}

// tc_retire (reading A8'): wait for and retire only the work enqueued before the previous retirement point — the
// work of this epoch keeps running.  tc_retire_lag (A8''): the lag-th previous point, so the last lag epochs keep
// running (lag 1 = tc_retire).
tc_status Pool::retire(int32_t lag) {
    if (lag < 1) return TC_E_INVAL;
    const uint32_t upto = epoch_id + 1 > (uint32_t)lag ? epoch_id + 1 - (uint32_t)lag : 0;
    if (!meta_only) {
        if (cuda_dead) return TC_E_CUDA;
        for (int32_t e : ev_used)
            if (ev_epoch[e] < upto) TC_CUDA(cudaEventSynchronize(events[e]), "retire wait");
    }
    retire_before(upto);
    return TC_OK;
}

// a4 / a7 bookkeeping for every pending entry, released slot, handle and event created before epoch `upto`, in
// issue order (A10); then a new epoch starts.  The caller has made sure that work has completed.
void Pool::retire_before(uint32_t upto) {
    size_t w = 0;
    for (size_t i = 0; i < pending_dev.size(); ++i) {
        if (pending_epoch[i] < upto) {
            const auto &pc = pending_dev[i];
            for (int32_t b : pc.second) {
                alloc.state[b] = kFree;
                alloc.set_free(b);
            }
            const int64_t k = (int64_t)pc.second.size();
            alloc.claimed[pc.first] -= std::min(k, alloc.claimed[pc.first]);
        } else {
            if (w != i) pending_dev[w] = std::move(pending_dev[i]);
            pending_epoch[w++] = pending_epoch[i];
        }
    }
    pending_dev.resize(w);
    pending_epoch.resize(w);
    // released slots back to their buffer
    for (size_t i = slots.released.size(); i-- > 0;) {
        if (slots.released_epoch[i] >= upto) continue;
        const int64_t x = slots.released[i];
        if (x < slots.count) {
            slots.give(x);
        } else if (is_peer(x)) {                           // peer-tier slot: back to its own free list
            peer.free_list.push_back(x);
        } else {
            auto sl = std::prev(extra.upper_bound(x));    // unbuffered ablation: free the slab with its last block
            if (--sl->second.live == 0) {
                if (sl->second.host) cudaFreeHost(sl->second.host);
                extra.erase(sl);
            }
        }
    }
    w = 0;
    for (size_t i = 0; i < slots.released.size(); ++i) {
        if (slots.released_epoch[i] < upto) continue;
        slots.released[w] = slots.released[i];
        slots.released_epoch[w++] = slots.released_epoch[i];
    }
    slots.released.resize(w);
    slots.released_epoch.resize(w);
    auto retired_ev = [&](int32_t e) { return e >= 0 && ev_epoch[e] < upto; };
    for (auto it = handles.begin(); it != handles.end();) {
        if (it->second.state == kUploaded && it->second.up_epoch < upto) {
            it = handles.erase(it);                        // B3: forgotten once its upload's epoch retires
        } else {
            if (retired_ev(it->second.ev)) it->second.ev = -1;
            ++it;
        }
    }
    for (auto &ag : agents)
        if (retired_ev(ag.up_event)) ag.up_event = -1;
    w = 0;
    for (size_t i = 0; i < ev_used.size(); ++i) {
        if (ev_epoch[ev_used[i]] < upto) {
            ev_free.push_back(ev_used[i]);
        } else {
            ev_used[w++] = ev_used[i];
        }
    }
    ev_used.resize(w);
    ++epoch_id;
}

tc_status Pool::fill(uint64_t seed) {
    if (meta_only) return TC_E_NODEV;
    if (cuda_dead) return TC_E_CUDA;
    TC_CUDA(launch_fill(kv, N, L, T, H, Hl, rank, D, seed, s_off), "fill kernel");
    ++n_launch;
    TC_CUDA(cudaStreamSynchronize(s_off), "fill sync");
    return TC_OK;
}

// ------------------------------------------------------------------------------------------------ per-call trace
static void CUDART_CB trace_done(void *rec) {
    reinterpret_cast<tc_trace_t *>(rec)->t_done_ns = steady_ns();
}

// One record per handle of a just-enqueued batch; their completion is stamped by a host callback queued on `s`
// behind the batch's work (so t_done - t_enqueued is the transfer as the host sees it).
void Pool::trace_calls(int32_t op, const int32_t *ags, const tc_handle *hs, const int64_t *off, int32_t k,
                       cudaStream_t s) {
    if (trace_cap <= 0) return;
    const int64_t t_enq = steady_ns();
    for (int32_t i = 0; i < k && trace_n < trace_cap; ++i) {
        tc_trace_t &r = trace_buf[trace_n++];
        const int64_t nb = off[i + 1] - off[i];
        r = tc_trace_t{op, ags ? ags[i] : handles.at(hs[i]).agent, hs[i], nb, nb * B, trace_t0, t_enq, 0};
        if (meta_only || cudaLaunchHostFunc(s, trace_done, &r) != cudaSuccess) {
            cudaGetLastError();
            r.t_done_ns = t_enq;
        }
    }
}

// TC_CHECK=1 (debug): the SPEC invariants re-derived from scratch after every mutating call;
// a violation aborts with the failing invariant.  Off by default (O(N) per call).
void Pool::check_descs(int32_t kind, const XferDesc *d, int64_t n) const {
    auto fail = [&](int64_t i, const char *what) {
        std::fprintf(stderr, "tokencake descriptor check failed (launch kind %d, descriptor %lld of %lld): %s\n", kind,
                     (long long)i, (long long)n, what);
        std::abort();
    };
    auto inside = [&](uint64_t x, const char *base, int64_t bytes) {
        const uint64_t b = reinterpret_cast<uint64_t>(base);
        return base && x >= b && x + (uint64_t)B <= b + (uint64_t)bytes;
    };
    const int64_t tab_n = (int64_t)max_agents * max_bpa;
    for (int64_t i = 0; i < n; ++i) {
        if (d[i].blk < 0 || d[i].blk >= N) fail(i, "pool block id out of range");
        if (d[i].tab < -1 || d[i].tab >= tab_n) fail(i, "block-table index out of range");
        const uint64_t x = d[i].ext;
        if (x % 16) fail(i, "block image not 16-byte aligned");
        bool ok = true;
        if (kind == 0 || kind == 1) {            // staged kernels: inside the direction's staging buffer
            ok = inside(x, staging[kind], staging_bytes);
        } else if (kind == 7 || kind == 8) {     // DIRECT kernels: a host slot of the slab or of an ablation slab
            ok = inside(x, slots.dev, slots.count * B);
            for (const auto &kv_ : extra)
                ok = ok || inside(x, kv_.second.dev, kv_.second.n * B);
        } else if (kind == 5 || kind == 6) {     // peer tier: the neighbour's slab
            ok = inside(x, peer.dev, peer.count * B);
        }                                        // kind 2: a caller buffer (the caller owns its extent)
        if (!ok) fail(i, "block image outside the buffer this launch may touch");
    }
}

void Pool::check_invariants(const char *after) const {
    auto fail = [&](const char *what) {
        std::fprintf(stderr, "tokencake invariant violated after %s: %s\n", after, what);
        std::abort();
    };
    int64_t nf = 0, na = 0, np = 0, nr = 0;
    for (int64_t b = 0; b < N; ++b) {
        const uint8_t st = alloc.state[b];
        const bool bit = (alloc.bits[b >> 6] >> (b & 63)) & 1;
        if (bit != (st == kFree)) fail("free bitmap != block state");
        nf += st == kFree; na += st == kAlloc; np += st == kPending; nr += st == kReserved;
    }
    if (nf + na + np + nr != N) fail("block conservation (S:113)");
    if (nf != alloc.nfree) fail("free count");
    if (nr != n_reserved) fail("reserved-block count");
    int64_t pend = 0;
    for (const auto &pc : pending_dev) pend += (int64_t)pc.second.size();
    if (pend != np) fail("pending list != PENDING blocks (P:648)");
    int64_t owned = 0;
    for (int32_t a = 0; a < max_agents; ++a) {
        const AgentRec &ag = agents[a];
        if (!ag.exists) continue;
        for (size_t pos = 0; pos < ag.table.size(); ++pos) {
            const int32_t b = ag.table[pos];
            if (b < 0) continue;
            ++owned;
            if (b >= N || alloc.state[b] != kAlloc || alloc.own_agent[b] != a || alloc.own_pos[b] != (int32_t)pos)
                fail("table <-> owner bijection");
        }
    }
    if (owned != na) fail("ALLOC blocks not all in tables");
    for (size_t c = 0; c < alloc.claimed.size(); ++c)
        if (alloc.claimed[c] < 0) fail("negative claim");
    if (!unbuffered) {
        int64_t host_in_use = 0, peer_in_use = 0, rel_host = 0, rel_peer = 0;
        for (const auto &hk : handles) {
            if (hk.second.state != kOffloaded) continue;
            for (int64_t s : hk.second.slots) (is_peer(s) ? peer_in_use : host_in_use) += 1;
        }
        for (int64_t s : slots.released) (is_peer(s) ? rel_peer : rel_host) += 1;
        if (slots.nfree + host_in_use + rel_host != slots.count) fail("host slot conservation");
        int64_t nb = 0;
        for (uint64_t x : slots.bits) nb += __builtin_popcountll(x);
        if (nb != slots.nfree) fail("host free set != free count");
        if ((int64_t)peer.free_list.size() + peer_in_use + rel_peer != peer.count) fail("peer slot conservation");
    }
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
    const bool foreign = s && s != s_off && s != s_up;
    cudaEvent_t fe = nullptr;
    if (foreign) {                  // tc_sync also waits for this launch: an event behind it, not the stream itself
        if (fev_free.empty()) {
            TC_CUDA(cudaEventCreateWithFlags(&fe, cudaEventDisableTiming), "caller-stream event");
            fev_free.push_back(fe);
        }
        fev_live.reserve(fev_live.size() + 1);
    }
    tc_status st = enqueue_xfer(gather, TC_XFER_DIRECT, desc, {}, s ? s : s_off);
    if (st != TC_OK || !foreign) return st;
    fe = fev_free.back();
    TC_CUDA(cudaEventRecord(fe, s), "caller-stream event");
    fev_free.pop_back();
    fev_live.push_back(fe);
    return TC_OK;
}

// Waits for every device-tier launch made on a caller stream since the last drain.
tc_status Pool::drain_foreign() {
    for (cudaEvent_t e : fev_live) TC_CUDA(cudaEventSynchronize(e), "sync caller-stream work");
    fev_free.insert(fev_free.end(), fev_live.begin(), fev_live.end());
    fev_live.clear();
    return TC_OK;
}

}  // namespace tc
