"""Where a kernel's CUDA-event span exceeds its own %globaltimer duration (GPU box): the device-tier gather (the staged
kernel, variant 3) of 1 / 8 / 64 / 256 MiB, timed (a) by its stamps, (b) by events around ONE launch on an idle
stream, (c) by events around K back-to-back launches (the per-launch excess of a busy stream), (d) with the stream
pre-loaded by a sleep kernel so the launch is already queued when the first event fires.  Prints JSON rows.
Tuning aid only."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T, N = 28, 4, 128, 16, 4096


def main():
    p = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=16)
    p.fill(3)
    B = p.block_bytes
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    rng = np.random.default_rng(1)
    dst = torch.empty(300 * B, dtype=torch.uint8, device=dev)
    for mib in (1, 8, 64, 256):
        n = max(1, (mib << 20) // B)
        ids = rng.choice(N, size=n, replace=False).astype(np.int32)

        def fn():
            p.gather_dev(ids, dst.data_ptr(), s.cuda_stream)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        p.sync()
        row = {"mib": round(n * B / 2**20, 1), "blocks": n}
        for mode in ("one_idle", "k8_busy", "one_preloaded"):
            spans, stamps = [], []
            for _ in range(10):
                p.timing(2)
                p.timing(2)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k = 8 if mode == "k8_busy" else 1
                if mode == "one_preloaded":
                    with torch.cuda.stream(s):
                        torch.cuda._sleep(2_000_000)      # ~1 ms: the launch below is queued before e0 fires
                e0.record(s)
                for _ in range(k):
                    fn()
                e1.record(s)
                e1.synchronize()
                p.sync()
                ms, cnt, _ = p.timing(0)["dev_device_kernel"]
                spans.append(e0.elapsed_time(e1) / k)
                stamps.append(ms / max(cnt, 1))
            row[mode + "_event_us"] = round(statistics.median(spans) * 1e3, 2)
            row[mode + "_stamp_us"] = round(statistics.median(stamps) * 1e3, 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
