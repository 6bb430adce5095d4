"""Can the copy engines do the device-side gather too? (GPU box; feasibility probe for a zero-SM staged path.)
C3-shaped blocks (2L = 64 chunks of 32 KiB, chunk pitch N*C in the layer-major pool): per block one strided 2-D
device-to-device cudaMemcpy2DAsync (pool -> contiguous staging slot), 256 blocks per batch.  Measures (1) that D2D
gather alone, (2) beside a host-link D2H + H2D pair on other streams, (3) a bf16 GEMM loop's slowdown beside the
CE gather + D2H loop vs beside the SM (TMA) gather + D2H loop.  Prints JSON lines; tuning aid only."""
import json
import os
import sys
import time

import numpy as np
import torch
from cuda.bindings import runtime as cudart

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T = 32, 8, 128, 16
N, NB = 4096, 256


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert int(err) == 0, r
    return r


def main():
    dev = torch.device("cuda", 0)
    p = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=16)
    p.fill(1)
    C, B = p.chunk_bytes, p.block_bytes
    kv = p.kv_ptr()
    stg = torch.empty(NB * B, dtype=torch.uint8, device=dev)
    ids = np.random.default_rng(3).choice(N, size=NB, replace=False)
    s = torch.cuda.Stream(dev)
    sp = s.cuda_stream
    D2D = cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice

    def ce_gather(stream=sp):
        for i, b in enumerate(ids):
            ck(cudaMemcpy2DAsync(stg.data_ptr() + i * B, C, kv + int(b) * C, N * C, C, 2 * L, D2D, stream))

    cudaMemcpy2DAsync = cudart.cudaMemcpy2DAsync
    # (1) alone
    ce_gather()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        ce_gather()
        host_ms = (time.perf_counter() - t0) * 1e3
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(json.dumps({"probe": "ce_2d_gather_alone", "bytes": NB * B, "ms": ms, "gbs_rw": 2 * NB * B / (ms * 1e-3) / 1e9,
                      "host_enqueue_ms": host_ms}), flush=True)
    # (2) beside host-link traffic
    hb = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    hb2 = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    db = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    db2 = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    with torch.cuda.stream(s1):
        for _ in range(4):
            hb.copy_(db, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(4):
            db2.copy_(hb2, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ce_gather()
    e1.record(s)
    e1.synchronize()
    ms2 = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    print(json.dumps({"probe": "ce_2d_gather_beside_link", "ms": ms2, "gbs_rw": 2 * NB * B / (ms2 * 1e-3) / 1e9}),
          flush=True)
    # (3) GEMM slowdown: CE gather -> D2H loop vs the library's SM gather (device tier, TMA) -> D2H loop
    n = 8192
    a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    bm = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    c = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    gs = torch.cuda.Stream(dev)
    iters = 300

    def gemms():
        with torch.cuda.stream(gs):
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(gs)
            for _ in range(iters):
                torch.matmul(a, bm, out=c)
            g1.record(gs)
        return g0, g1
    g0, g1 = gemms()
    torch.cuda.synchronize()
    alone = g0.elapsed_time(g1)
    hbuf = torch.empty(NB * B, dtype=torch.uint8, pin_memory=True)
    for name in ("ce_gather", "sm_gather"):
        g0, g1 = gemms()
        moved = 0
        t0 = time.perf_counter()
        while not g1.query():
            if name == "ce_gather":
                ce_gather()
            else:
                p.gather_dev(ids.astype(np.int32), stg.data_ptr(), sp)
            with torch.cuda.stream(s):
                hbuf.copy_(stg, non_blocking=True)
            s.synchronize()
            moved += NB * B
        secs = time.perf_counter() - t0
        torch.cuda.synchronize()
        print(json.dumps({"probe": "gemm_beside_" + name + "_d2h", "gemm_slowdown": g0.elapsed_time(g1) / alone,
                          "offload_gbs": moved / secs / 1e9}), flush=True)
    p.sync()


if __name__ == "__main__":
    main()
