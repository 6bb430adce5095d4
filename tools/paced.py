"""Paced Time-Scheduler loop on the GPU (SURVEY.md §8(d) "paced mode"): agents alternate LLM phases and function calls
in wall-clock time; at each call's start the NEXT-3 decision layer (Eq. 1 forecast + EWMA, Alg. 1 ShouldOffload with
T_transfer calibrated from this pool's own transfers) decides whether to offload the agent's KV blocks, and the
predictive-upload plan issues the upload so that it lands before the predicted return.  At the call's
real return the agent needs its blocks: the time it waits for them is the stall (an early return triggers an
immediate upload).

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
    stats = {ag: (None, 0) for ag in range(a.agents)}   # per-agent EWMA history (t_hist, n_obs)
    ev = []                                            # (time_s, seq, kind, agent, payload)
    seq = 0

    def push(t, kind, ag, payload=None):
        nonlocal seq
        heapq.heappush(ev, (t, seq, kind, ag, payload))
        seq += 1

    t0 = time.perf_counter()
    for ag in range(a.agents):
        push(t0 + rng.exponential(a.llm_mean_ms) / 1e3, "fc_start", ag)
    live = {}                                          # agent -> dict(handle, upload_issued, call_end)
    stalls, lateness, decisions, freed_block_s, transfers = [], [], {"offload": 0, "retain": 0}, 0.0, 0
    end = t0 + a.seconds
    while ev:
        t, _, kind, ag, payload = heapq.heappop(ev)
        if t > end and kind == "fc_start":
            continue
        now = time.perf_counter()
        if t > now:
            time.sleep(t - now)
        now = time.perf_counter()
        if kind == "fc_start":
            n = sizes[ag]
            d_true = rng.exponential(a.fc_mean_ms)
            t_hist, n_obs = stats[ag]
            t_fc = sched.fc_predict(t_hist, n_obs, cold_start=a.fc_mean_ms)
            t_tr = sched.transfer_ms(n, model["offload_ms_per_block"], model["upload_ms_per_block"])
            waiting = [n * cfg.T * 0.5]                 # a waiting request of half the freed tokens
            dec = sched.should_offload(n, t_fc, t_tr, a.v_tok_s, waiting)
            call_end = now + d_true / 1e3
            if dec["offload"]:
                decisions["offload"] += 1
                h = pool.offload(ag, pool.block_table(ag))
                off_ms = n * model["offload_ms_per_block"]
                up_ms = n * model["upload_ms_per_block"]
                plan = sched.plan_upload(0.0, t_fc, up_ms, off_ms)
                live[ag] = {"h": h, "issued": False, "t_off": now, "t_up": None}
                push(now + max(plan["upload_start"], off_ms) / 1e3, "upload", ag)
            else:
                decisions["retain"] += 1
            push(call_end, "fc_end", ag, d_true)
        elif kind == "upload":
            st = live.get(ag)
            if st and not st["issued"]:
                pool.upload(st["h"])
                st["issued"], st["t_up"] = True, now
        elif kind == "fc_end":
            d_true = payload
            st = live.pop(ag, None)
            if st is not None:
                if not st["issued"]:                    # early return: immediate prefetch
                    pool.upload(st["h"])
                    st["t_up"] = now
                try:
                    pool.wait(st["h"])
                except tcb.TcError as e:                # already retired by an earlier tc_sync: it has landed
                    if e.status != tcb.E_HANDLE:
                        raise
                ready = time.perf_counter()
                stalls.append((ready - t) * 1e3)        # from the call's true return (includes loop lateness)
                lateness.append((now - t) * 1e3)
                freed_block_s += sizes[ag] * ((st["t_up"] or now) - st["t_off"])
                transfers += 2
                pool.sync()                             # retire the pending source blocks and released slots
            stats[ag] = sched.fc_observe(stats[ag][0], stats[ag][1], d_true)
            push(time.perf_counter() + rng.exponential(a.llm_mean_ms) / 1e3, "fc_start", ag)
    wall = time.perf_counter() - t0
    pool.sync()
    zero = sum(1 for s in stalls if s < 0.25)      # below the loop's own wake-up + tc_wait cost
    out = {
        "what": "paced Time-Scheduler loop (Eq. 1 + EWMA, Alg. 1, predictive upload) on C2-shaped KV, 1 x B200",
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
        "transfers": transfers,
    }
    print(json.dumps(out), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/paced_{int(a.fc_mean_ms)}ms.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
