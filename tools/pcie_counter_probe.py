"""Host-link counters (NVML, the GPU's own PCIe byte counters) while one tc_cycle after another moves a C2-shaped
batch both ways, per transfer path pair — the question being whether DIRECT uploads (SM reads of mapped host
memory) leave the link idle (a per-request-stream cap on outstanding reads) or fill it with protocol overhead.

Per path pair (d2h/h2d = staged|direct): the payload rate each direction from the pool's own byte counts and the
loop's CUDA-event time, and the PCIe TX (out of the GPU) / RX (into the GPU) bytes over the same interval from NVML:
the cumulative counters (NVML_FI_DEV_PCIE_COUNT_TX/RX_BYTES) when the driver exposes them, and the 20 ms throughput
samples (nvmlDeviceGetPcieThroughput) always; plus the link's replay / NAK counters.  The wire carries the payload
plus TLP headers and, for reads, request TLPs in the other direction: an SM-read-bound upload shows RX well below
the copy engine's while TX (its read requests + the D2H payload) stays put.

    python tools/pcie_counter_probe.py [--blocks 256] [--seconds 3]
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

F_TX, F_RX = pynvml.NVML_FI_DEV_PCIE_COUNT_TX_BYTES, pynvml.NVML_FI_DEV_PCIE_COUNT_RX_BYTES
F_REPLAY, F_NAK_R, F_NAK_S = (pynvml.NVML_FI_DEV_PCIE_REPLAY_COUNTER, pynvml.NVML_FI_DEV_PCIE_COUNT_NAKS_RECEIVED,
                              pynvml.NVML_FI_DEV_PCIE_COUNT_NAKS_SENT)


def fields(h, ids):
    """{field id: value or None} (None: not supported by this driver / VM)."""
    out = {}
    try:
        vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
    except pynvml.NVMLError:
        return {i: None for i in ids}
    for i, v in zip(ids, vals):
        if v.nvmlReturn != 0:
            out[i] = None
            continue
        out[i] = {0: v.value.dVal, 1: v.value.uiVal, 2: v.value.ulVal, 3: v.value.ullVal,
                  4: v.value.sllVal}.get(v.valueType, v.value.ullVal)
    return out


class Sampler(threading.Thread):
    """nvmlDeviceGetPcieThroughput every `dt` s (KB/s averaged over the driver's 20 ms window)."""

    def __init__(self, h, dt=0.02):
        super().__init__(daemon=True)
        self.h, self.dt, self.stop_ev, self.tx, self.rx = h, dt, threading.Event(), [], []

    def run(self):
        while not self.stop_ev.is_set():
            try:
                self.tx.append(pynvml.nvmlDeviceGetPcieThroughput(self.h, pynvml.NVML_PCIE_UTIL_TX_BYTES) * 1e3)
                self.rx.append(pynvml.nvmlDeviceGetPcieThroughput(self.h, pynvml.NVML_PCIE_UTIL_RX_BYTES) * 1e3)
            except pynvml.NVMLError:
                pass
            time.sleep(self.dt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=256)
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    L, H, D = 28, 4, 128                      # C2 geometry: 1.75 MiB block shards
    NB = a.blocks
    p = tcb.Pool(L, H, D, 16, "bf16", 4 * NB + 64, device=0, host_slots=3 * NB + 16, max_blocks_per_agent=4 * NB)
    p.fill(3)
    for ag in (0, 1, 2):
        p.agent_add(ag, 0)
    for _ in range(NB):                       # scattered ids: three agents grown interleaved
        for ag in (0, 2, 1):
            p.alloc(ag, 1)
    p.sync()
    B = p.block_bytes
    up_s, off_s = p.streams()
    ups = torch.cuda.ExternalStream(up_s, device=0)
    offs = torch.cuda.ExternalStream(off_s, device=0)
    modes = {"staged": tcb.XFER_STAGED, "direct": tcb.XFER_DIRECT}
    for d2h, h2d in (("staged", "staged"), ("direct", "staged"), ("staged", "direct"), ("direct", "direct")):
        p.set_xfer_mode(modes[d2h], modes[h2d])
        hnd = p.offload(0, p.block_table(0))  # agent 0 on the host; agent 1 resident
        p.sync()
        on_host, on_dev = 0, 1

        def cycle():
            nonlocal hnd, on_host, on_dev
            _, out = p.cycle([hnd], [(on_dev, p.block_table(on_dev))])
            hnd = out[0]
            on_host, on_dev = on_dev, on_host

        for _ in range(3):                    # warm-up
            cycle()
            p.retire(1)
        p.sync()
        c0 = fields(h, [F_TX, F_RX, F_REPLAY, F_NAK_R, F_NAK_S])
        smp = Sampler(h)
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e0[0].record(ups)
        e0[1].record(offs)
        smp.start()
        t0, n = time.perf_counter(), 0
        while time.perf_counter() - t0 < a.seconds:
            cycle()
            p.retire(1)
            n += 1
        p.sync()
        e1[0].record(ups)
        e1[1].record(offs)
        torch.cuda.synchronize()
        smp.stop_ev.set()
        smp.join()
        c1 = fields(h, [F_TX, F_RX, F_REPLAY, F_NAK_R, F_NAK_S])
        secs = max(e0[0].elapsed_time(e1[0]), e0[1].elapsed_time(e1[1])) * 1e-3
        pay = n * NB * B                       # bytes each way
        row = {"d2h": d2h, "h2d": h2d, "cycles": n, "blocks_per_cycle": NB, "block_bytes": B, "seconds": round(secs, 3),
               "payload_gbs_each_way": round(pay / secs / 1e9, 2), "payload_gbs_both": round(2 * pay / secs / 1e9, 2)}
        for key, f in (("tx", F_TX), ("rx", F_RX)):
            if c0[f] is not None and c1[f] is not None:
                row[f"pcie_{key}_gbs_counter"] = round((c1[f] - c0[f]) / secs / 1e9, 2)
        trim = lambda xs: xs[len(xs) // 10: len(xs) - len(xs) // 10] or xs  # noqa: E731  (drop ramp samples)
        if smp.tx:
            row["pcie_tx_gbs_sampled_median"] = round(statistics.median(trim(smp.tx)) / 1e9, 2)
            row["pcie_rx_gbs_sampled_median"] = round(statistics.median(trim(smp.rx)) / 1e9, 2)
            row["samples"] = len(smp.tx)
        for key, f in (("replays", F_REPLAY), ("naks_received", F_NAK_R), ("naks_sent", F_NAK_S)):
            if c0[f] is not None and c1[f] is not None:
                row[key] = c1[f] - c0[f]
        print(json.dumps(row), flush=True)
        p.sync()
        p.upload(hnd)                          # back to both agents resident for the next pair
        p.sync()
    p.close()
    pynvml.nvmlShutdown()


if __name__ == "__main__":
    main()
