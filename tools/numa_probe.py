"""Host NUMA placement of pinned memory on the GPU box: node count, the GPU's local CPUs / node, and the node of
sampled pages of a pinned (cudaHostAlloc) buffer allocated after bench.py's CPU binding (move_pages(2), no libnuma).

    python tools/numa_probe.py [GiB]
"""
import ctypes
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def nodes():
    out = {}
    for d in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        n = int(d.rsplit("node", 1)[1])
        cpus = open(os.path.join(d, "cpulist")).read().strip()
        mem = [l for l in open(os.path.join(d, "meminfo")) if "MemFree" in l or "MemTotal" in l]
        out[n] = (cpus, [" ".join(l.split()[2:4]) for l in mem])
    return out


def page_nodes(addr, nbytes, samples=4096):
    libc = ctypes.CDLL(None, use_errno=True)
    page = os.sysconf("SC_PAGE_SIZE")
    step = max(page, (nbytes // samples) // page * page)
    ptrs = [addr + i * step for i in range(nbytes // step)]
    n = len(ptrs)
    arr = (ctypes.c_void_p * n)(*ptrs)
    status = (ctypes.c_int * n)()
    SYS_move_pages = 279
    r = libc.syscall(SYS_move_pages, 0, ctypes.c_ulong(n), arr, None, status, 0)
    if r != 0:
        return {"error": ctypes.get_errno()}
    hist = {}
    for s in status:
        hist[s] = hist.get(s, 0) + 1
    return hist


def main():
    import torch
    import bench
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    print("nodes:", nodes())
    print("binding:", bench.bind_numa_local(0))
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        cands = glob.glob("/sys/bus/pci/devices/*" + bus.lower()[-10:] + "/numa_node")
        print("gpu0 pci", bus, "numa_node", [open(c).read().strip() for c in cands])
    except Exception as e:  # noqa: BLE001
        print("nvml:", e)
    t = torch.empty(int(gib * (1 << 30)), dtype=torch.uint8, pin_memory=True)
    print(f"pinned {gib} GiB page nodes (status -> count):", page_nodes(t.data_ptr(), t.numel()))
    import paper_2510_18586_b200 as tcb
    from workloads.configs import CONFIGS
    cfg = CONFIGS["c2"]
    pool = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, 4096, device=0, host_slots=cfg.host_slots(),
                    max_agents=64, max_blocks_per_agent=4096)
    pool.agent_add(0, 0)
    pool.alloc(0, 8)
    h = pool.offload(0, pool.block_table(0))
    pool.sync()
    vp = ctypes.c_void_p()
    pool._check(tcb.lib.tc_handle_host(pool._h, h, 0, ctypes.byref(vp)))
    ptr = vp.value                                   # slot 0 = the slab's base (first pop of the LIFO)
    print("library slab first slot ptr:", ptr)
    if ptr:
        print("library slab page nodes (10 GiB from the first offloaded slot):",
              page_nodes(ptr, min(cfg.host_slots() * pool.block_bytes, 10 << 30)))


if __name__ == "__main__":
    main()
