// Host-memory read probe (GPU box; a measurement tool, not part of the library): why SM-issued reads of mapped pinned
// memory slow down while the other link direction is busy ("The DIRECT kernels").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hostread_probe tools/hostread_probe.cu && /tmp/hostread_probe
//
// 1. latency: one thread chases a random pointer chain through mapped pinned host memory (one 4 KiB page per hop,
//    so every hop is a fresh PCIe read), %globaltimer per hop;
// 2. throughput: CTAs x 256 threads stream 16-byte loads from mapped host memory (kUnroll in flight per thread);
// each alone, beside a copy-engine D2H stream (the other direction busy, as in a DIRECT upload next to a staged
// offload) and beside a copy-engine H2D stream (the same direction busy).  Little's law then says how many bytes the
// SMs keep in flight: throughput x latency.  Prints one JSON object per line.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void chase(const uint64_t *__restrict__ base, uint64_t start, int hops, unsigned long long *out) {
    uint64_t idx = start;
    const unsigned long long t0 = gtime();
    for (int i = 0; i < hops; ++i) idx = *(volatile const uint64_t *)(base + idx);
    const unsigned long long t1 = gtime();
    out[0] = t1 - t0;
    out[1] = idx;   // keep the chain live
}

constexpr int kUnroll = 8;
__global__ void stream_read(const int4 *__restrict__ src, int64_t n_vec, int4 *__restrict__ sink,
                            unsigned long long *ts) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMin(ts, gtime());
    int4 acc = make_int4(0, 0, 0, 0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kUnroll;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; v < n_vec; v += stride) {
        int4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t k = v + (int64_t)u * blockDim.x;
            r[u] = k < n_vec ? src[k] : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) acc.x ^= r[u].x, acc.y ^= r[u].y, acc.z ^= r[u].z, acc.w ^= r[u].w;
    }
    if (acc.x == 0x7fffffff) sink[threadIdx.x] = acc;   // practically never: keeps the loads
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(ts + 1, gtime());
}

// background SM writes into mapped host memory (the DIRECT D2H kernel's traffic), `reps` passes over the buffer
__global__ void stream_write(int4 *__restrict__ dst, int64_t n_vec, int reps) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vec; v += stride)
            dst[v] = make_int4(r, (int)v, 0, 0);
}

int main() {
    CK(cudaSetDevice(0));
    const size_t chain_bytes = 256ull << 20, page = 4096;
    const size_t nodes = chain_bytes / page;
    uint64_t *hchain = nullptr, *dchain = nullptr;
    CK(cudaHostAlloc((void **)&hchain, chain_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer((void **)&dchain, hchain, 0));
    std::vector<uint64_t> perm(nodes);
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin() + 1, perm.end(), std::mt19937_64(7));
    const uint64_t words = page / 8;
    for (size_t i = 0; i < nodes; ++i) hchain[perm[i] * words] = perm[(i + 1) % nodes] * words;

    const size_t rd_bytes = 1ull << 30;
    int4 *hread = nullptr, *dread = nullptr;
    CK(cudaHostAlloc((void **)&hread, rd_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer((void **)&dread, hread, 0));
    std::memset(hread, 1, rd_bytes);
    // background copy-engine traffic
    const size_t bg_bytes = 1ull << 30;
    void *bg_host = nullptr, *bg_dev = nullptr;
    CK(cudaHostAlloc(&bg_host, bg_bytes, cudaHostAllocPortable | cudaHostAllocMapped));
    CK(cudaMalloc(&bg_dev, bg_bytes));
    int4 *sink = nullptr;
    unsigned long long *dts = nullptr;
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMalloc(&dts, 64));
    cudaStream_t sk, sb;
    CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    cudaEvent_t bg_done, k_done;
    CK(cudaEventCreate(&bg_done));
    CK(cudaEventCreate(&k_done));

    int4 *bg_host_mapped = nullptr;
    CK(cudaHostGetDevicePointer((void **)&bg_host_mapped, bg_host, 0));
    const char *bg_names[4] = {"alone", "beside_ce_d2h", "beside_ce_h2d", "beside_sm_d2h"};
    for (int bg = 0; bg < 4; ++bg) {
        auto start_bg = [&]() {   // ~24 GiB of background traffic, longer than any measurement below
            if (bg == 3) {
                stream_write<<<74, 256, 0, sb>>>(bg_host_mapped, (int64_t)(bg_bytes / 16), 24);
                CK(cudaGetLastError());
            }
            for (int i = 0; i < 24 && (bg == 1 || bg == 2); ++i)
                CK(cudaMemcpyAsync(bg == 1 ? bg_host : bg_dev, bg == 1 ? bg_dev : bg_host, bg_bytes,
                                   bg == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, sb));
            CK(cudaEventRecord(bg_done, sb));
        };
        // latency
        start_bg();
        const int hops = 20000;
        unsigned long long hres[2];
        chase<<<1, 1, 0, sk>>>(dchain, 0, 2000, dts);          // warm
        chase<<<1, 1, 0, sk>>>(dchain, perm[nodes / 2] * words, hops, dts);
        CK(cudaEventRecord(k_done, sk));
        CK(cudaEventSynchronize(k_done));   // the background must still be running when the kernel ends
        const bool overlapped = cudaEventQuery(bg_done) == cudaErrorNotReady || bg == 0;
        CK(cudaEventSynchronize(bg_done));
        CK(cudaMemcpy(hres, dts, 16, cudaMemcpyDeviceToHost));
        std::printf("{\"probe\": \"latency\", \"traffic\": \"%s\", \"ns_per_hop\": %.1f, \"overlapped\": %s}\n",
                    bg_names[bg], (double)hres[0] / hops, overlapped ? "true" : "false");
        // throughput per grid size
        for (int ctas : {4, 8, 16, 32, 74, 148, 296}) {
            unsigned long long init[2] = {~0ull, 0};
            CK(cudaMemcpy(dts, init, 16, cudaMemcpyHostToDevice));   // before the background starts
            start_bg();
            const int64_t n_vec = (int64_t)(rd_bytes / 16);
            stream_read<<<ctas, 256, 0, sk>>>(dread, n_vec, sink, dts);
            CK(cudaEventRecord(k_done, sk));
            CK(cudaEventSynchronize(k_done));
            const bool ov = cudaEventQuery(bg_done) == cudaErrorNotReady || bg == 0;
            CK(cudaEventSynchronize(bg_done));
            CK(cudaMemcpy(hres, dts, 16, cudaMemcpyDeviceToHost));
            const double ns = (double)(hres[1] - hres[0]);
            const double inflight = (double)ctas * 256 * kUnroll * 16;
            std::printf("{\"probe\": \"read\", \"traffic\": \"%s\", \"ctas\": %d, \"bytes_in_flight_max\": %.0f, "
                        "\"gbs\": %.2f, \"overlapped\": %s}\n",
                        bg_names[bg], ctas, inflight, rd_bytes / ns, ov ? "true" : "false");
        }
    }
    return 0;
}
