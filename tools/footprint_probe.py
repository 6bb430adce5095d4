"""Host-link rate vs the pinned host footprint the copies walk through (is the bench loop's H2D shortfall against the
1 GiB best-of-10 link probe a property of the host side — IOMMU / host DRAM — rather than of the loop?).

For a pinned slab of S GiB (cudaHostAlloc through torch pin_memory) and device buffers of 1 GiB per direction:
  fixed    both directions copy 1 GiB at the same host offsets every rep (what bench.py's hostlink_peak does)
  walk     each rep uses the next 1 GiB of its half of the slab (the whole slab is touched, like the host slots)
  runs     each rep moves 1 GiB as R-MiB contiguous runs at shuffled slab offsets (the loop's DMA-run pattern)
Each line: mode, per-direction GB/s inside the concurrent pair and the pair's total, best and median of `reps`.

    python tools/footprint_probe.py [slab_GiB=16] [reps=8] [run_MiB=64] [alloc=torch|lib]

alloc=lib allocates the slab as libtokencake does (cudaHostAlloc Portable | Mapped) instead of torch's pin_memory.
"""
import json
import random
import statistics
import sys

import torch


def main():
    slab_gib = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    run_mib = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    alloc = sys.argv[4] if len(sys.argv) > 4 else "torch"
    G = 1 << 30
    dev = torch.device("cuda:0")
    if alloc == "lib":                                     # the library's CPU block buffer allocation
        import ctypes
        torch.cuda.init()
        rt = ctypes.CDLL("libcudart.so.12")
        ptr = ctypes.c_void_p()
        assert rt.cudaHostAlloc(ctypes.byref(ptr), ctypes.c_size_t(slab_gib * G), 1 | 2) == 0   # Portable|Mapped
        buf = (ctypes.c_uint8 * (slab_gib * G)).from_address(ptr.value)
        host = torch.frombuffer(buf, dtype=torch.uint8)
        assert host.is_pinned()
    else:
        host = torch.empty(slab_gib * G, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)                                          # first touch: every page backed before timing
    d_up = torch.empty(G, dtype=torch.uint8, device=dev)
    d_off = torch.empty(G, dtype=torch.uint8, device=dev)
    d_off.fill_(2)
    s_up, s_off = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    half = slab_gib // 2
    rng = random.Random(7)

    def pair(up_pieces, off_pieces):
        """up_pieces / off_pieces: lists of (host byte offset, device byte offset, nbytes)."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        ev[0].record(s_up)
        ev[2].record(s_off)
        with torch.cuda.stream(s_up):
            for h, d, n in up_pieces:
                d_up[d:d + n].copy_(host[h:h + n], non_blocking=True)
        with torch.cuda.stream(s_off):
            for h, d, n in off_pieces:
                host[h:h + n].copy_(d_off[d:d + n], non_blocking=True)
        ev[1].record(s_up)
        ev[3].record(s_off)
        torch.cuda.synchronize()
        t_up, t_off = ev[0].elapsed_time(ev[1]) * 1e-3, ev[2].elapsed_time(ev[3]) * 1e-3
        return G / t_up / 1e9, G / t_off / 1e9, 2 * G / max(t_up, t_off) / 1e9

    def runs(base_gib, k):
        R = run_mib << 20
        n = G // R
        slots = list(range(half * G // R))
        rng.shuffle(slots)
        return [(base_gib * G + s * R, i * R, R) for i, s in enumerate(slots[:n])]

    modes = {
        "fixed": lambda k: ([(0, 0, G)], [(half * G, 0, G)]),
        "walk": lambda k: ([((k % half) * G, 0, G)], [((half + k % half) * G, 0, G)]),
        "runs": lambda k: (runs(0, k), runs(half, k)),
    }
    for name, f in modes.items():
        pair(*f(0))                                        # warm-up
        res = [pair(*f(k)) for k in range(reps)]
        out = {"mode": name, "alloc": alloc, "slab_gib": slab_gib, "run_mib": run_mib if name == "runs" else None, "reps": reps}
        for i, key in enumerate(("h2d_gbs", "d2h_gbs", "pair_gbs")):
            xs = [r[i] for r in res]
            out[key] = {"best": round(max(xs), 2), "median": round(statistics.median(xs), 2)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
