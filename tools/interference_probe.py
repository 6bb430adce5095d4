"""Transfers beside model compute (GPU box): the offload/upload path runs while the serving engine's kernels keep the
SMs busy (the transfers are asynchronous to inference).  A bf16 GEMM loop (8192^3, cuBLAS, on its own
stream) stands in for the model; C3-shaped offload + upload cycles (256 blocks = 512 MiB each way per cycle) run on
the library's streams at the same time.  Per transfer configuration: the GEMM loop's TFLOP/s beside the transfers vs
alone, and the transfers' GB/s beside the GEMMs vs alone.

Configurations: STAGED with the default device-side grid (whole waves of 296+ CTAs, 96 KiB smem each), STAGED with
a 32-CTA device-side grid (the gather / scatter still finish far ahead of their DMA), DIRECT both ways (the SMs move
the bytes for the whole transfer), direct D2H + staged H2D.  Prints JSON lines; tuning aid, the bench is bench.py.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T = 32, 8, 128, 16          # C3 block shard: 2 MiB
NB = 256


def gemm_loop(a, b, c, iters, stream):
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            torch.matmul(a, b, out=c)
        e1.record(stream)
    return e0, e1


def main():
    dev = torch.device("cuda", 0)
    n = 8192
    a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    c = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    gs = torch.cuda.Stream(dev)
    iters = int(os.environ.get("IP_ITERS", 300))
    # GEMM alone
    e0, e1 = gemm_loop(a, b, c, 20, gs)
    torch.cuda.synchronize()
    e0, e1 = gemm_loop(a, b, c, iters, gs)
    torch.cuda.synchronize()
    alone_ms = e0.elapsed_time(e1)
    flops = 2.0 * n ** 3 * iters
    print(json.dumps({"gemm_alone_tflops": flops / (alone_ms * 1e-3) / 1e12, "ms": alone_ms}), flush=True)

    configs = [("staged_default", tcb.XFER_STAGED, tcb.XFER_STAGED, (0, 32, 3)),
               ("staged_32ctas", tcb.XFER_STAGED, tcb.XFER_STAGED, (32, 32, 3)),
               ("direct_both", tcb.XFER_DIRECT, tcb.XFER_DIRECT, (0, 32, 3)),
               ("direct_d2h_staged_h2d", tcb.XFER_DIRECT, tcb.XFER_STAGED, (0, 32, 3))]
    for name, d2h, h2d, dev_cfg in configs:
        p = tcb.Pool(L, H, D, T, "bf16", 4 * NB + 64, device=0, host_slots=3 * NB, xfer_d2h=d2h, xfer_h2d=h2d,
                     max_blocks_per_agent=4 * NB)
        p.set_launch_config(2, *dev_cfg)
        p.fill(1)
        p.agent_add(0, 0)
        p.agent_add(1, 0)
        for _ in range(NB):
            p.alloc(0, 1)
            p.alloc(1, 1)
        B = p.block_bytes
        h = p.offload(0, p.block_table(0))
        p.sync()

        def cycles(k):
            nonlocal h
            moved = 0
            t0 = time.perf_counter()
            on = 1
            for _ in range(k):
                _, hs = p.cycle([h], [(on, p.block_table(on))])
                p.retire(1)
                h = hs[0]
                on ^= 1
                moved += 2 * NB * B
            p.sync()
            return moved, time.perf_counter() - t0

        cycles(2)
        moved, secs = cycles(10)                      # transfers alone
        alone_gbs = moved / secs / 1e9
        torch.cuda.synchronize()
        e0, e1 = gemm_loop(a, b, c, iters, gs)        # GEMMs queued; transfers run beside them
        moved2, secs2 = 0, 0.0
        t0 = time.perf_counter()
        while not e1.query():
            m, s = cycles(2)
            moved2 += m
        secs2 = time.perf_counter() - t0
        torch.cuda.synchronize()
        beside_ms = e0.elapsed_time(e1)
        print(json.dumps({"config": name, "transfer_alone_gbs": alone_gbs,
                          "transfer_beside_gemm_gbs": moved2 / secs2 / 1e9 if secs2 else None,
                          "gemm_beside_tflops": flops / (beside_ms * 1e-3) / 1e12,
                          "gemm_slowdown": beside_ms / alone_ms}), flush=True)
        p.upload(h)
        p.sync()
        p.close()


if __name__ == "__main__":
    main()
