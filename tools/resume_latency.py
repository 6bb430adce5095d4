"""When can each agent of a cycle resume?  C3 scheduling cycles (8 uploads + 8 offloads of ~290 blocks, 2 MiB block
shards) through tc_cycle; for every upload handle a side stream waits on it (tc_stream_wait — what an engine's decode
of that agent would do) and records an event: the agent's resume time from the cycle's start.  Per-handle completion
events (default) vs batch-granular (TC_FINE_DEPS=0 in the environment).  Each cycle is drained before the next, so
the numbers are per cycle, not pipelined.

    [TC_FINE_DEPS=0] python tools/resume_latency.py [cycles=12]
Prints one JSON row: ms from the cycle's start to the 1st / median / last agent's resume (p50 over cycles).
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402
from workloads.scripts import CycleGen, setup_ops  # noqa: E402


def main():
    n_cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    cfg = CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    p = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, cfg.N, device=0, host_slots=cfg.host_slots(),
                 max_agents=1024, max_blocks_per_agent=cfg.max_blocks_per_agent)
    p.fill(cfg.seed)
    ops, agents, _ = setup_ops(cfg)
    for op in ops:
        getattr(p, {"reserve": "reserve", "agent_add": "agent_add", "alloc": "alloc", "agent_free": "agent_free",
                    "sync": "sync"}[op[0]])(*op[1:])
    gen = CycleGen(cfg, agents, combined=True)
    handles = {}
    up_s, _ = p.streams()
    ups = torch.cuda.ExternalStream(up_s, device=dev)
    sides = [torch.cuda.Stream(dev) for _ in range(cfg.per_cycle)]
    rows = []
    for cyc in range(n_cycles + 3):
        for op in gen.next_cycle():
            if op[0] != "cycle":
                continue
            hs = [handles.pop(a) for a in op[1]]
            offs = [(a, [b for b in p.block_table(a) if b >= 0]) for a, _ in op[2]]
            p.sync()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(ups)
            _, out_h = p.cycle(hs, offs)
            evs = []
            for h, st in zip(hs, sides):
                p.stream_wait(h, st.cuda_stream)
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                evs.append(e)
            for (a, _), h in zip(offs, out_h):
                handles[a] = h
            torch.cuda.synchronize(dev)
            if cyc >= 3 and evs:
                t = sorted(e0.elapsed_time(e) for e in evs)
                rows.append((t[0], t[len(t) // 2], t[-1]))
    p.sync()
    print(json.dumps({"fine_deps": os.environ.get("TC_FINE_DEPS", "1") != "0", "cycles": len(rows),
                      "uploads_per_cycle": cfg.per_cycle,
                      "first_ms": round(statistics.median(r[0] for r in rows), 2),
                      "median_ms": round(statistics.median(r[1] for r in rows), 2),
                      "last_ms": round(statistics.median(r[2] for r in rows), 2)}))
    p.close()


if __name__ == "__main__":
    main()
