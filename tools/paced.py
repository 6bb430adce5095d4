"""Paced Time-Scheduler loop on the GPU (SURVEY.md §8(d) "paced mode"): agents alternate LLM phases and function calls
in wall-clock time, and the native Time Scheduler (tc_ts_*, csrc/sched.cpp) decides at each call's start whether to
offload the agent's KV blocks (Eq. 1 forecast + EWMA, Alg. 1 ShouldOffload with T_transfer calibrated from this pool's
own transfers), reserves destination blocks gradually and issues the upload from its scheduling ticks so that it lands
before the predicted return.  At the call's real return the agent needs its blocks: the time it waits
for them is the stall (an early return triggers an immediate upload).

Workload: C2 geometry (Qwen2.5-7B-shaped 896 KiB block shards), 16 agents with C2's log-normal sizes; function-call
durations ~ Exp(mean) per agent class (Table 1 "short" tools: 100 ms), LLM phases ~ Exp(50 ms); a waiting
request whose demand fits is always present, so Alg. 1 offloads whenever the window beats the transfer.
Prints one JSON summary and writes gpurun_out/paced_<mean>ms.json.

  python tools/paced.py [--seconds 15] [--fc-mean-ms 100]
"""
import argparse
import heapq
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from paper_2510_18586_b200 import sched  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402
from workloads.scripts import agent_sizes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=15.0)
    ap.add_argument("--fc-mean-ms", type=float, default=100.0)
    ap.add_argument("--llm-mean-ms", type=float, default=50.0)
    ap.add_argument("--agents", type=int, default=16)
    ap.add_argument("--tick-ms", type=float, default=5.0)
    ap.add_argument("--lead-ms", type=float, default=10.0)
    ap.add_argument("--v-tok-s", type=float, default=20000.0,
                    help="engine decode throughput (tokens/s) for Alg. 1's N_capacity")
    a = ap.parse_args()
    cfg = CONFIGS["c2"]
    rng = np.random.default_rng(cfg.seed)
    sizes = agent_sizes(cfg.scaled(N=cfg.N), rng)[:a.agents]
    N = 4 * sum(sizes) + 256
    pool = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, N, device=0, host_slots=2 * sum(sizes) + 64,
                    max_blocks_per_agent=max(sizes) + 8)
    pool.fill(cfg.seed)
    pool.timing(1)                                  # link-side spans feed tc_xfer_model_measure (calibration)
    for ag, n in enumerate(sizes):
        pool.agent_add(ag, ag % 3)
        pool.alloc(ag, n)
    # calibrate T_transfer with one warm-up round trip per agent
    for ag in range(a.agents):
        h = pool.offload(ag, pool.block_table(ag))
        pool.sync()
        pool.upload(h)
        pool.sync()
    model = sched.xfer_model_measure(pool)
    ts = sched.TimeScheduler(pool, model=model, v_tokens_per_s=a.v_tok_s, cold_start_ms=a.fc_mean_ms,
                             tick_ms=a.tick_ms, reserve_cycles=4, lead_ms=a.lead_ms)
    ev = []                                            # (time_s, seq, kind, agent, payload)
    seq = 0

    def push(t, kind, ag, payload=None):
        nonlocal seq
        heapq.heappush(ev, (t, seq, kind, ag, payload))
        seq += 1

    t0 = time.perf_counter()
    ms = lambda t: (t - t0) * 1e3                      # the engine clock handed to the scheduler  # noqa: E731
    for ag in range(a.agents):
        push(t0 + rng.exponential(a.llm_mean_ms) / 1e3, "fc_start", ag)
    push(t0, "tick", -1)
    stalls, lateness, decisions, offload_t, freed_block_s = [], [], {"offload": 0, "retain": 0}, {}, 0.0
    end = t0 + a.seconds
    while ev:
        t, _, kind, ag, payload = heapq.heappop(ev)
        if t > end and kind in ("fc_start", "tick"):
            continue
        now = time.perf_counter()
        if t > now:
            time.sleep(t - now)
        now = time.perf_counter()
        if kind == "tick":                             # the engine's scheduling tick: reservations + due uploads
            ts.tick(ms(now))
            push(t + a.tick_ms / 1e3, "tick", -1)
        elif kind == "fc_start":
            d_true = rng.exponential(a.fc_mean_ms)
            waiting = [sizes[ag] * cfg.T * 0.5]         # a waiting request of half the freed tokens
            dec = ts.call_start(ag, 0, ms(now), waiting=waiting)
            decisions["offload" if dec["offload"] else "retain"] += 1
            if dec["offload"]:
                offload_t[ag] = now
            push(now + d_true / 1e3, "fc_end", ag, d_true)
        elif kind == "fc_end":
            h = ts.call_finish(ag, ms(now))            # issues the upload now if the plan had not yet
            if h:
                try:
                    pool.wait(h)
                except tcb.TcError as e:                # already retired by an earlier tc_sync: it has landed
                    if e.status != tcb.E_HANDLE:
                        raise
                ready = time.perf_counter()
                stalls.append((ready - t) * 1e3)        # from the call's true return (includes loop lateness)
                lateness.append((now - t) * 1e3)
                freed_block_s += sizes[ag] * (now - offload_t.pop(ag))
                pool.sync()                             # retire the pending source blocks and released slots
            push(time.perf_counter() + rng.exponential(a.llm_mean_ms) / 1e3, "fc_start", ag)
    wall = time.perf_counter() - t0
    pool.sync()
    zero = sum(1 for s in stalls if s < 0.25)      # below the loop's own wake-up + tc_wait cost
    out = {
        "what": "paced loop driving the native Time Scheduler (tc_ts_*: Eq. 1 + EWMA, Alg. 1, gradual reservation, "
                "predictive upload) on C2-shaped KV, 1 x B200",
        "agents": a.agents, "fc_mean_ms": a.fc_mean_ms, "llm_mean_ms": a.llm_mean_ms, "seconds": wall,
        "xfer_model": model, "calls": decisions["offload"] + decisions["retain"], **decisions,
        "stall_ms": {"p50": statistics.median(stalls) if stalls else None,
                     "p99": float(np.percentile(stalls, 99)) if stalls else None,
                     "max": max(stalls) if stalls else None,
                     "zero_stall_frac": zero / len(stalls) if stalls else None,
                     "event_loop_lateness_p50": statistics.median(lateness) if lateness else None,
                     "how": "agent's wait for its blocks after the call's true return, offloaded calls only"},
        "kv_block_seconds_freed": freed_block_s,
        "avg_blocks_off_gpu": freed_block_s / wall,
        "avg_kv_gib_off_gpu": freed_block_s / wall * pool.block_bytes / 2**30,
        "transfers": 2 * len(stalls),
    }
    print(json.dumps(out), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/paced_{int(a.fc_mean_ms)}ms.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
