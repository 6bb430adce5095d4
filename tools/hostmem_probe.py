"""Pinned host memory backing vs host-link bandwidth: one buffer from cudaHostAlloc (torch pin_memory) and one from
mmap + madvise(MADV_HUGEPAGE) + first touch + cudaHostRegister; for each, H2D alone, D2H alone and both directions
concurrently (1 GiB each way, best of 5), and the share of the buffer backed by transparent huge pages.

    python tools/hostmem_probe.py [GiB]
"""
import ctypes
import json
import mmap
import sys

import torch

libc = ctypes.CDLL(None, use_errno=True)
MADV_HUGEPAGE = 14


def thp_kib(addr, nbytes):
    """AnonHugePages (kB) of the smaps entries overlapping [addr, addr + nbytes)."""
    tot, inside = 0, False
    for line in open("/proc/self/smaps"):
        f = line.split()
        if "-" in f[0] and len(f[0]) > 8 and all(c in "0123456789abcdef-" for c in f[0]):
            a, b = (int(x, 16) for x in f[0].split("-"))
            inside = a < addr + nbytes and b > addr
        elif inside and f[0] == "AnonHugePages:":
            tot += int(f[1])
    return tot


def bench(host, dev, reps=5):
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    n = host.numel()

    def t(fn):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    half = n // 2
    h2d = n / (t(lambda: dev[:n].copy_(host, non_blocking=True)) * 1e-3) / 1e9

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            dev[:half].copy_(host[:half], non_blocking=True)
        with torch.cuda.stream(s2):
            host[half:].copy_(dev[half:n], non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    d2h = n / (t(lambda: host.copy_(dev[:n], non_blocking=True)) * 1e-3) / 1e9
    bi = n / (t(both) * 1e-3) / 1e9
    return {"h2d": h2d, "d2h": d2h, "bidir": bi}


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    n = int(gib * (1 << 30))
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    a.fill_(1)
    out["cudaHostAlloc"] = dict(bench(a, dev), thp_mib=thp_kib(a.data_ptr(), n) / 1024)
    del a
    m = mmap.mmap(-1, n + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    addr = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    r = libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(n), MADV_HUGEPAGE)
    ctypes.memset(addr, 1, n)
    cr = torch.cuda.cudart().cudaHostRegister(addr, n, 0)
    buf = (ctypes.c_uint8 * n).from_address(addr)
    h = torch.frombuffer(buf, dtype=torch.uint8)
    out["mmap_thp_register"] = dict(bench(h, dev), thp_mib=thp_kib(addr, n) / 1024, madvise=r, register=int(cr))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
