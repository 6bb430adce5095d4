"""The bench loop's DMA pattern without the library (GPU box): both directions stream P-MiB pieces continuously for
~2 s between a 16 GiB pinned slab (allocated as libtokencake does: cudaHostAlloc Portable | Mapped) and two device
staging halves per direction — optionally with a device-to-device copy of each piece on a third stream standing in
for the gather / scatter kernels' HBM traffic.  Per direction: GB/s over the streaming interval.  Compare with the
1 GiB best-of-10 probe (bench.py hostlink_peak) on the same box: if this pattern alone shows the loop's H2D shortfall,
the shortfall is the DMA pattern (piece size, footprint), not the library's kernels or events.

    python tools/dma_pattern_probe.py
Prints JSON rows.  Tuning aid only.
"""
import ctypes
import json

import torch


def main():
    G = 1 << 30
    slab_gib = 16
    dev = torch.device("cuda:0")
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    ptr = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(ptr), ctypes.c_size_t(slab_gib * G), 1 | 2) == 0
    host = torch.frombuffer((ctypes.c_uint8 * (slab_gib * G)).from_address(ptr.value), dtype=torch.uint8)
    host.fill_(3)
    stg_up = torch.empty(G, dtype=torch.uint8, device=dev)       # two 512 MiB halves per direction
    stg_off = torch.empty(G, dtype=torch.uint8, device=dev)
    pool = torch.empty(4 * G, dtype=torch.uint8, device=dev)
    import os
    hi = os.environ.get("PROBE_UP_PRIORITY") == "1"             # the library's upload streams run at high priority
    s_up = torch.cuda.Stream(dev, priority=-1 if hi else 0)
    s_off, s_k = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    half = slab_gib // 2 * G

    def run(piece_mib, kernels, secs=2.0, pingpong=False):
        P = piece_mib << 20
        n = int(secs * 50e9 / P) + 1                            # pieces per direction for ~secs at 50 GB/s
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        ev[0].record(s_up)
        ev[2].record(s_off)
        for i in range(n):
            hb = (i * P) % (half - P)
            db = (i % 2) * (G // 2)
            seg = min(P, G // 2)
            if pingpong:                                        # upload what the offload wrote k pieces earlier
                k = 8
                src = half + ((i - k) * P) % (half - P) if i >= k else hb
                with torch.cuda.stream(s_up):
                    stg_up[db:db + seg].copy_(host[src:src + seg], non_blocking=True)
            else:
                with torch.cuda.stream(s_up):                   # upload: slab -> staging half
                    stg_up[db:db + seg].copy_(host[hb:hb + seg], non_blocking=True)
            with torch.cuda.stream(s_off):                      # offload: staging half -> slab (other half)
                host[half + hb:half + hb + seg].copy_(stg_off[db:db + seg], non_blocking=True)
            if kernels:                                         # HBM traffic of a gather + a scatter per piece
                with torch.cuda.stream(s_k):
                    pool[:seg].copy_(stg_up[db:db + seg], non_blocking=True)
                    stg_off[db:db + seg].copy_(pool[G:G + seg], non_blocking=True)
        ev[1].record(s_up)
        ev[3].record(s_off)
        torch.cuda.synchronize()
        up = n * min(P, G // 2) / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9
        off = n * min(P, G // 2) / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9
        return {"piece_mib": piece_mib, "kernels": kernels, "pingpong": pingpong, "pieces": n, "h2d_gbs": round(up, 2),
                "d2h_gbs": round(off, 2), "both_gbs": round(up + off, 2)}

    run(512, False, 0.5)                                        # warm-up
    for piece in (512, 128, 32):
        for k in (False, True):
            print(json.dumps(run(piece, k)), flush=True)
    for k in (False, True):                                     # uploads of recently offloaded host memory
        print(json.dumps(run(512, k, pingpong=True)), flush=True)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench                                                # the bench's own link probe, same box, same call
    r = bench.hostlink_peak(torch, dev)
    print(json.dumps({"hostlink_peak": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()
                                        if k != "how"}}))


if __name__ == "__main__":
    main()
