"""B200 analogue of the paper's Fig. 11 (fig:evo_transfer_overhead): offload / upload latency for
1,024-5,120 blocks with and without the overhead mitigations (CPU Block Buffering P:475-484, Gradual GPU Block
Reservation P:486-495).  NEXT-1 row of SURVEY.md §8(f).

Arms: "unbuffered" (tc_pool_desc.unbuffered: cudaHostAlloc per offload, cudaFreeHost at retirement; all-at-once
device allocation), "buffered" (CPU block buffer; all-at-once allocation) and "buffered+gradual" (CPU block buffer;
destination blocks claimed over 4 ticks before the upload).  For each: host call-return latency of tc_offload /
tc_upload and completion latency (call -> tc_wait returns).  Block = C2's 896 KiB shard (Qwen2.5-7B-shaped).
Writes gpurun_out/fig11.json.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T = 28, 4, 128, 16
SIZES = [int(x) for x in os.environ.get("FIG11_SIZES", "1024,2048,3072,4096,5120").split(",")]
N = 2 * max(SIZES) + 64
REPS = int(os.environ.get("FIG11_REPS", 3))


def run_arm(unbuffered, gradual):
    p = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=max(SIZES) + 8, unbuffered=unbuffered,
                 max_blocks_per_agent=max(SIZES) + 8)
    p.fill(11)
    p.agent_add(0, 0)
    p.agent_add(1, 1)
    rows = []
    for n in SIZES:
        for rep in range(REPS + 1):
            ids = p.alloc(0, n)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = p.offload(0, ids)
            t1 = time.perf_counter()
            p.wait(h)
            t2 = time.perf_counter()
            p.sync()
            if gradual:
                p.reserve_begin(h, 4)
                for _ in range(4):
                    p.reserve_tick()
            t3 = time.perf_counter()
            new = p.upload(h)
            t4 = time.perf_counter()
            p.wait(h)
            t5 = time.perf_counter()
            p.sync()                             # unbuffered: the per-offload pinned slab is freed here
            t6 = time.perf_counter()
            p.agent_free(0)
            p.sync()
            if rep:
                rows.append({"blocks": n, "bytes": n * p.block_bytes,
                             "offload_call_ms": (t1 - t0) * 1e3, "offload_done_ms": (t2 - t0) * 1e3,
                             "upload_call_ms": (t4 - t3) * 1e3, "upload_done_ms": (t5 - t3) * 1e3,
                             "retire_ms": (t6 - t5) * 1e3})
            assert len(new) == n
    p.close()
    out = []
    for n in SIZES:
        r = [x for x in rows if x["blocks"] == n]
        out.append({k: (float(np.median([x[k] for x in r])) if k not in ("blocks", "bytes") else r[0][k])
                    for k in r[0]})
    return out


def main():
    res = {"block_bytes": 2 * L * T * H * D * 2, "sizes": SIZES, "reps": REPS}
    for name, ub, gr in (("buffered+gradual", False, True), ("buffered", False, False), ("unbuffered", True, False)):
        res[name] = run_arm(ub, gr)
        for row in res[name]:
            print(name, json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/fig11.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
