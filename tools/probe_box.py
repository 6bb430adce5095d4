"""Box probe: host-link (PCIe) roofline via pinned cudaMemcpyAsync.

Writes gpurun_out/hostlink.json. Plumbing measurement only (torch copies), no product code.
"""
import json, os, subprocess, time
import torch

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return str(e)

def bw(fn, nbytes, reps=10):
    best = 0.0
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        best = max(best, nbytes / (s.elapsed_time(e) * 1e-3) / 1e9)
    return best

def main():
    out = {"nvidia_smi": sh("nvidia-smi"), "topo": sh("nvidia-smi topo -m"), "numa": sh("numactl -H; lscpu"),
           "mem": sh("free -g"), "cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
           "driver": sh("nvidia-smi --query-gpu=driver_version,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current --format=csv")}
    dev = torch.device("cuda:0")
    res = {}
    for size in [1 << 20, 8 << 20, 64 << 20, 256 << 20, 1 << 30]:
        h = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(size, dtype=torch.uint8, device=dev)
        d2 = torch.empty(size, dtype=torch.uint8, device=dev)
        h2d = bw(lambda: d.copy_(h, non_blocking=True), size)
        d2h = bw(lambda: h.copy_(d, non_blocking=True), size)
        s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
        def bidir():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur); s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            cur.wait_stream(s1); cur.wait_stream(s2)
        bi = bw(bidir, 2 * size)
        res[str(size)] = {"h2d_gbs": h2d, "d2h_gbs": d2h, "bidir_total_gbs": bi}
        print(size, res[str(size)], flush=True)
        del h, h2, d, d2
    out["hostlink"] = res
    # pinned alloc cost
    t = time.perf_counter(); x = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True); out["pin_4GiB_s"] = time.perf_counter() - t
    del x
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/hostlink.json", "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k in ("hostlink", "pin_4GiB_s", "cpu_count", "affinity")}, indent=1))
    print(out["topo"]); print(out["driver"]); print(out["mem"])

if __name__ == "__main__":
    main()
