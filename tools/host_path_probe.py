"""Host cost of one small scheduling cycle (GPU box): tc_cycle of k blocks up + k blocks off (C5 G = 8 shard geometry,
640 KiB blocks), per transfer mode — the library call's host time (median / p90 of `reps` calls, from Python, so it
includes the ctypes marshalling) and the completion time (call -> both handles complete).  With TC_HOST_TRACE=1 the
library also prints, per cycle, the host microseconds at which each enqueue step returned.

    python tools/host_path_probe.py [reps=400]
Tuning aid; prints JSON rows.
"""
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    L, H, D, G = 80, 8, 128, 8
    N = 4096
    for mode_name, mode in (("direct", tcb.XFER_DIRECT), ("staged", tcb.XFER_STAGED), ("auto", tcb.XFER_AUTO)):
        for k in (1, 8):
            p = tcb.Pool(L, H, D, 16, "bf16", N, device=0, shard_world=G, host_slots=256, xfer_d2h=mode,
                         xfer_h2d=mode)
            p.fill(1)
            for a in (0, 1):
                p.agent_add(a, 0)
                p.alloc(a, k)
            h = p.offload(0, p.block_table(0))
            p.sync()
            on_dev = 1
            call, done = [], []
            for r in range(reps + 20):
                hs = np.array([h], dtype=np.uint64)
                uoff = np.array([0, k], dtype=np.int64)
                ags = np.array([on_dev], dtype=np.int32)
                ids = np.ascontiguousarray(p.block_table_np(on_dev))
                ooff = np.array([0, len(ids)], dtype=np.int64)
                t0 = time.perf_counter()
                _, out_h = p.cycle_arrays(hs, uoff, ags, ooff, ids)
                t1 = time.perf_counter()
                p.wait(int(out_h[0]))
                p.wait(int(h))
                t2 = time.perf_counter()
                if r >= 20:
                    call.append((t1 - t0) * 1e6)
                    done.append((t2 - t0) * 1e6)
                h = int(out_h[0])
                on_dev ^= 1
                p.retire(1)
            p.sync()
            q = lambda xs, f: round(float(np.percentile(xs, f)), 1)  # noqa: E731
            print(json.dumps({"mode": mode_name, "blocks": k, "block_bytes": p.block_bytes, "reps": reps,
                              "call_us_p50": round(statistics.median(call), 1), "call_us_p90": q(call, 90),
                              "done_us_p50": round(statistics.median(done), 1), "done_us_p90": q(done, 90)}),
                  flush=True)
            p.close()


if __name__ == "__main__":
    main()
