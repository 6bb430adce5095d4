"""Offload / upload latency and throughput vs blocks per offload (BASELINE configs[4]: C5 "sweep 1-512 blocks per
offload"), one direction at a time, per transfer mode.  Block = one rank's shard of the config (C5: G = 8, 640 KiB).

For each size s and mode: REPS offloads of s physically scattered blocks (two agents grown interleaved, so ids
alternate), then their uploads; per call the host call-return time and the completion time (call -> tc_wait
returns), p50 / p99, and the completion-time throughput.  Writes gpurun_out/sweep_<cfg>.json.

  python tools/sweep.py [c5] [--modes staged,direct]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402

MODES = {"staged": tcb.XFER_STAGED, "direct": tcb.XFER_DIRECT, "copy": tcb.XFER_COPY}


def pct(x, q):
    return float(np.percentile(np.asarray(x), q))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--modes", default="staged,direct")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    G = cfg.G if a.config == "c5" else 1
    sizes = list(cfg.sweep) or [1, 4, 16, 64, 256]
    smax = max(sizes)
    N = 4 * smax + 64
    res = {"config": a.config, "head_shards": G, "sizes": sizes, "reps": a.reps, "rows": []}
    for mname in a.modes.split(","):
        m = MODES[mname]
        p = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, N, device=0, shard_world=G, host_slots=2 * smax + 8,
                     max_blocks_per_agent=2 * smax + 8, xfer_d2h=m, xfer_h2d=m)
        p.fill(cfg.seed)
        B = p.block_bytes
        p.agent_add(0, 0)
        p.agent_add(1, 1)
        for _ in range(smax):                       # interleaved growth: agent 0's ids are every other block
            p.alloc(0, 1)
            p.alloc(1, 1)
        for s in sizes:
            rows = {"off_call": [], "off_done": [], "up_call": [], "up_done": []}
            for rep in range(a.reps + 2):
                ids = p.block_table(0)[:s]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                h = p.offload(0, ids)
                t1 = time.perf_counter()
                p.wait(h)
                t2 = time.perf_counter()
                p.sync()
                t3 = time.perf_counter()
                p.upload(h)
                t4 = time.perf_counter()
                p.wait(h)
                t5 = time.perf_counter()
                p.sync()
                if rep >= 2:
                    rows["off_call"].append((t1 - t0) * 1e3)
                    rows["off_done"].append((t2 - t0) * 1e3)
                    rows["up_call"].append((t4 - t3) * 1e3)
                    rows["up_done"].append((t5 - t3) * 1e3)
            r = {"mode": mname, "blocks": s, "bytes": s * B}
            for k, v in rows.items():
                r[k + "_p50_ms"] = statistics.median(v)
                r[k + "_p99_ms"] = pct(v, 99)
            r["off_gbs"] = s * B / (r["off_done_p50_ms"] * 1e-3) / 1e9
            r["up_gbs"] = s * B / (r["up_done_p50_ms"] * 1e-3) / 1e9
            res["rows"].append(r)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
        p.close()
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/sweep_{a.config}.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
