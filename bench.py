#!/usr/bin/env python
"""Benchmark of the Tokencake offload/upload hot path on B200 (one process per GPU).

A *step* is one scheduling cycle of the whole hot path through the C ABI, in the
P:645-648 order: the cycle's uploads of agents whose function call is over (a5 allocation + a6 H2D scatter with the
fused table remap), then the cycle's offloads of agents entering a function call (a2 admission + a3 gather/D2H), then
its retirement point (a4, a7).  By default the retirement is tc_retire_lag(k) — the transfers enqueued before the
k-th previous point return their blocks and slots while the last k cycles stream on, the asynchronous loop of
P:645-648 (readings A8', A8''; k = the largest <= 4 the host buffer and free blocks carry, from the warm-up cycles);
--retire sync drains every cycle with tc_sync instead (that number is also reported, as `per_cycle_drain`).

  python bench.py [--gpus N --steps K --warmup W] [--workload c2|c3|c4|c5] [--mode auto|direct|staged]
  python bench.py --impl reference ...     # the CPU oracle (oracle/), timed on the host cores

--gpus N > 1 without a torchrun environment re-launches itself as N ranks (torch.distributed.run, 127.0.0.1), one
process per GPU.  Default workload: at N = 1, C3 (BASELINE.json configs[2], Llama-3-8B-shaped KV, Deep-Research-style
64 agents with Space-Scheduler partitions: the largest single-GPU config); at N > 1, C4 head-sharded with G = N (the
north_star's KV-head partition: each GPU moves its own head shard of every block through its own host link; strong
scaling).  --workload c2 / c3 run independent pools per rank (weak), --workload c5 one rank's G = 8 shard per GPU
(weak) plus the 1-512 blocks-per-offload sweep.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads.configs import CONFIGS  # noqa: E402
from workloads.scripts import CycleGen, setup_ops  # noqa: E402

METRIC = "KV offload/upload GB/s and blocks/s per GPU vs host-link & HBM peak at 1/2/4/8 GPUs"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
XFER_NAMES = {1: "direct", 2: "staged", 3: "copy"}
NVLINK_GBS = 770.0      # peer copy per direction, measured on this pool (B200_PROFILING.md; 900 nominal)
HBM_FALLBACK = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback (GB/s), only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None)
    ap.add_argument("--mode", default="auto", choices=["auto", "direct", "staged", "copy", "mixed", "mixed_rev"],
                    help="transfer path per direction; mixed = direct D2H + staged H2D, mixed_rev = the reverse")
    ap.add_argument("--peer", action="store_true",
                    help="NEXT-2 peer tier: as many peer slots as host slots, in the next GPU's HBM (this GPU's own "
                         "HBM when it is alone); offloads go there first")
    ap.add_argument("--trace", default=None, metavar="FILE",
                    help="write the per-call trace (tc_trace) of the diagnostic steps as JSONL")
    ap.add_argument("--retire", default="auto", choices=["auto", "each", "sync"],
                    help="each: every step is tc_cycle + tc_retire (retire the previous cycle's transfers without "
                         "draining this one's: the asynchronous loop of P:645-648); sync: tc_cycle + tc_sync "
                         "(drain every step); auto: each, with the lag the warm-up cycles show the host buffer and "
                         "free blocks can carry (a refused cycle is retried after tc_retire, then after tc_sync)")
    ap.add_argument("--retire-lag", type=int, default=0,
                    help="retire-each loop: tc_retire_lag(lag) — retire what was enqueued before the lag-th previous "
                         "point, so lag cycles stay in flight; 0 = auto: the largest lag <= 4 whose in-flight host "
                         "slots and blocks fit (judged from the warm-up cycles)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--quick", action="store_true", help="skip the host-link probes (before and after), the device-tier microbench and the resume probe")
    ap.add_argument("--no-sweep", action="store_true", help="c5: skip the 1-512 blocks-per-offload sweep")
    ap.add_argument("--head-shards", type=int, default=0,
                    help="c4 on one GPU: run one rank's shard of a G-GPU head-sharded run (G = 1, 2, 4, 8) — the work "
                         "each GPU of that run does, alone on this GPU and its own host link (per-GPU flatness)")
    ap.add_argument("--shard-rank", type=int, default=0, help="with --head-shards: which rank's shard (0 .. G-1)")
    ap.add_argument("--host-frac", type=float, default=0.0,
                    help="pinned host slots as a fraction of N (default: the config's, 0.25 for C3-C5) — a study "
                         "knob: the paper's box had 100 GB of host swap per GPU (P:674)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rendezvous / workload-plan check without a GPU: every rank joins the process group "
                         "(gloo), rank 0 prints the plan line (n_gpus, head shards, per-rank rows, cpu_baseline)")
    return ap.parse_args()


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_command(argv: list, gpus: int, port: int) -> list:
    """The torchrun command bench.py re-executes itself with when --gpus N > 1 is given outside torchrun (the
    driver's own N > 1 launch line, loopback rendezvous)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(args, argv) -> int | None:
    """--gpus N > 1 with no WORLD_SIZE in the environment: run N ranks through torchrun and return its exit code
    (None = already inside a launcher, or a single GPU)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(launch_command(argv, args.gpus, free_port()), env=env)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def default_workload(world: int) -> str:
    """C3 on one GPU (the largest single-GPU config: 64 agents, Space-Scheduler quotas); the
    head-sharded C4 (G = N) on N > 1 GPUs — the north_star's KV-head partition."""
    return "c3" if world == 1 else "c4"


def shard_rank_for(args, rank, G):
    """This rank's head shard: rank mod G, or --shard-rank when one GPU runs one shard of a G-GPU run."""
    if getattr(args, "head_shards", 0):
        if not 0 <= args.shard_rank < G:
            raise SystemExit(f"--shard-rank must be in [0, {G})")
        return args.shard_rank
    return rank % G if G > 1 else 0


def workload_for(args, world):
    """(config, head shards G, scaling).  C4 is head-sharded over the ranks present (G = N: strong scaling; at N = 1
    the whole 128 GiB pool sits on one GPU).  C5 is defined on 8 x B200 (BASELINE configs[4]): G = 8 always, and N < 8
    GPUs run N of its 8 rank shards (80 GiB each) — fixed work per GPU, weak scaling.  C1-C3: one whole pool per
    rank, independent agent sets (weak)."""
    name = args.workload or default_workload(world)
    cfg = CONFIGS[name]
    hs = getattr(args, "head_shards", 0) or 0
    if hs:
        if name != "c4" or world != 1 or cfg.H % hs:
            raise SystemExit("--head-shards: c4 on one GPU (N = 1), G dividing its 8 KV heads")
        return cfg, hs, ("strong" if hs > 1 else "weak")
    if name == "c4":
        return cfg, world, ("strong" if world > 1 else "weak")
    if name == "c5":
        return cfg, cfg.G, "weak"
    return cfg, 1, "weak"


# ------------------------------------------------------------------------------------------------- measurement aids
class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.p = None
        if os.environ.get("TC_BENCH_CLOCKS") == "0":     # experiments only: no sampler
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out = self.p.communicate(timeout=5)[0]
        except Exception:  # noqa: BLE001
            self.p.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0])); smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def bind_numa_local(index: int) -> str:
    """Pin this rank's threads to the CPUs NVML reports as local to GPU `index`, before any pinned allocation, so the
    CPU block buffer (cudaHostAlloc, first touch) lands in the GPU's own NUMA node and each GPU's host traffic stays
    on its own socket's memory (matters at 8 GPUs; a no-op on a 1-socket box)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
        return f"{len(cpus)} cpus local to GPU {index}"
    except Exception as e:  # noqa: BLE001 - affinity is an optimisation, never a failure
        return f"unbound ({type(e).__name__})"


def hostlink_peak(torch, dev, nbytes=1 << 30, reps=10):
    """Pinned cudaMemcpyAsync D2H / H2D / bidirectional, best of `reps`."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def best(fn, nb):
        fn(); torch.cuda.synchronize(dev)
        b = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            b = max(b, nb / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        return b

    split = {"h2d": 0.0, "d2h": 0.0}

    def bidir():
        cur = torch.cuda.current_stream(dev)
        s1.wait_stream(cur); s2.wait_stream(cur)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s1); ev[2].record(s2)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        ev[1].record(s1); ev[3].record(s2)
        cur.wait_stream(s1); cur.wait_stream(s2)
        ev[3].synchronize(); ev[1].synchronize()
        split["h2d"] = max(split["h2d"], nbytes / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9)
        split["d2h"] = max(split["d2h"], nbytes / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9)

    r = {"h2d_gbs": best(lambda: d.copy_(h, non_blocking=True), nbytes),
         "d2h_gbs": best(lambda: h.copy_(d, non_blocking=True), nbytes),
         "bidir_gbs": best(bidir, 2 * nbytes), "bytes": nbytes, "how": "torch pinned copy_ 1 GiB, best of 10"}
    r["bidir_split_gbs"] = dict(split)          # each direction's own rate inside the concurrent pair (best)
    del h, h2, d, d2
    return r


def link_probe(torch, dev, dist, rank, world):
    """(alone, concurrent) host-link peaks of this rank: alone = measured while every other rank waits at a barrier;
    concurrent = all ranks measuring at once (the per-GPU denominator at N > 1).  At N = 1 they are one measurement."""
    alone = None
    for r in range(world):
        if dist is not None:
            dist.barrier()
        if r == rank:
            alone = hostlink_peak(torch, dev)
    if world == 1:
        return alone, alone
    dist.barrier()
    conc = hostlink_peak(torch, dev)
    dist.barrier()
    conc["how"] += ", all ranks concurrently"
    alone["how"] += ", this rank alone (the others at a barrier)"
    return alone, conc


def resume_probe(torch, dev, pool, cycle, ups, per_cycle, n=6):
    """When can each agent of a cycle resume?  n drained cycles after the timed region: a side stream per upload
    handle waits on it (tc_stream_wait, as an engine's decode of that agent would) and records an event; ms from the
    cycle's start (an event on the upload stream just before tc_cycle) to the first / median / last agent, p50."""
    sides = [torch.cuda.Stream(dev) for _ in range(max(1, per_cycle))]
    rows = []
    for _ in range(n):
        pool.sync()
        t0 = torch.cuda.Event(enable_timing=True)
        evs = []

        def rec(what):
            if what == "start":
                t0.record(ups)

        def on_up(hs):
            for h, st in zip(hs, sides):
                pool.stream_wait(int(h), st.cuda_stream)
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                evs.append(e)

        cycle(record=rec, retire="sync", on_uploads=on_up)
        torch.cuda.synchronize(dev)
        if evs:
            t = sorted(t0.elapsed_time(e) for e in evs)
            rows.append((t[0], t[len(t) // 2], t[-1]))
    if not rows:
        return None
    return {"first_ms": statistics.median(r[0] for r in rows), "median_ms": statistics.median(r[1] for r in rows),
            "last_ms": statistics.median(r[2] for r in rows), "cycles": len(rows),
            "how": "drained cycles after the timed region: per upload handle a side stream behind tc_stream_wait "
                   "records an event; ms from the cycle's start to the first / median / last agent's resume, p50"}


def offload_size_sweep(pool, cfg, B, sizes=None, reps=8):
    """C5's "sweep 1-512 blocks per offload" (BASELINE configs[4]; the Fig. 11 micro-benchmark): two
    sweep agents grown interleaved one block at a time (physically scattered ids); per size s and rep one tc_cycle
    uploads s blocks of the agent offloaded last rep while it offloads s blocks of the other — both directions
    concurrent — then the roles swap.  Per size: host call-return and completion (call -> both handles waited)
    latency p50 / p99, and GB/s = 2 s B / completion p50."""
    sizes = list(sizes or cfg.sweep or (1, 2, 4, 8, 16, 32, 64, 128, 256, 512))
    smax = max(sizes)
    pool.sync()
    X, Y = 1022, 1023
    for a in (X, Y):
        pool.agent_add(a, 7)                 # background class: outside the Space-Scheduler quotas
    for _ in range(smax):
        pool.alloc(X, 1)
        pool.alloc(Y, 1)
    pool.sync()
    rows = []
    for sz in sizes:
        h = pool.offload(Y, pool.block_table(Y)[:sz])
        pool.wait(h)
        pool.sync()
        on, off_agent = X, Y                 # `on` is on the GPU and offloads; `off_agent` uploads handle h
        call, done = [], []
        for rep in range(reps + 2):
            ids = pool.block_table(on)[:sz]
            t0 = time.perf_counter()
            _, hs = pool.cycle([h], [(on, ids)])
            t1 = time.perf_counter()
            pool.wait(h)
            pool.wait(hs[0])
            t2 = time.perf_counter()
            pool.sync()
            if rep >= 2:
                call.append((t1 - t0) * 1e3)
                done.append((t2 - t0) * 1e3)
            h, on, off_agent = hs[0], off_agent, on
        pool.upload(h)
        pool.sync()
        p50 = statistics.median(done)
        rows.append({"blocks": sz, "bytes_per_direction": sz * B,
                     "call_p50_ms": statistics.median(call), "call_p99_ms": float(np.percentile(call, 99)),
                     "done_p50_ms": p50, "done_p99_ms": float(np.percentile(done, 99)),
                     "gbs": 2 * sz * B / (p50 * 1e-3) / 1e9, "blocks_per_s": 2 * sz / (p50 * 1e-3)})
    for a in (X, Y):
        pool.agent_free(a)
    pool.sync()
    return {"rows": rows, "reps": reps, "block_shard_bytes": B,
            "how": "per size s: tc_cycle(upload s blocks of one sweep agent, offload s blocks of the other) — both "
                   "directions concurrent — from host arrays; call = host time of the tc_cycle call, done = call -> "
                   "tc_wait of both handles; GB/s = 2 s B / done p50 (both directions)"}


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "B200_PROFILING.md fallback"


def per_gpu_summary(rows) -> dict:
    """Per-rank throughput from rows [dev_ms, host_ms, bytes, blocks, wall_s(, link bidir GB/s concurrent)] (one per
    rank): own bytes / own device time, the spread across ranks (flat per GPU = small spread) and, when the rank's
    concurrently measured link peak is in the row, own GB/s as a fraction of it."""
    gbs = [r[2] / (r[0] * 1e-3) / 1e9 if r[0] else 0.0 for r in rows]
    bps = [r[3] / (r[0] * 1e-3) if r[0] else 0.0 for r in rows]
    mean = sum(gbs) / len(gbs)
    out = {"gbs": gbs, "blocks_per_s": bps, "min_gbs": min(gbs), "max_gbs": max(gbs), "mean_gbs": mean,
           "spread": (max(gbs) - min(gbs)) / mean if mean else None,
           "how": "per rank: own KV bytes / own device time of the timed region (all_gather); value = all ranks' "
                  "bytes / the max-over-ranks time"}
    if all(len(r) > 5 and r[5] for r in rows):
        out["link_bidir_gbs"] = [r[5] for r in rows]
        out["link_frac"] = [g / r[5] for g, r in zip(gbs, rows)]
    return out


def choose_retire(retire: str, retire_lag: int, host_free: int, free: int, up_max: int, off_max: int,
                  max_lag: int = 4) -> tuple[str, int]:
    """(retire mode, lag) for the timed loop, from the pool's free host slots / free blocks after the drained warm-up
    cycles and the warm-up's largest upload / offload cycle (blocks).  Retire-each with lag k keeps k more cycles of
    host slots (released by uploads) and of pending source blocks (offloads) unreturned than a drained loop does:
    it fits when host_free >= 1.1 (1 + k) off_max and free >= 1.1 (up_max + (1 + k) off_max) (10 % margin).
    auto -> each (a cycle the host buffer refuses takes the retire ladder: tc_retire, then tc_sync — so a loop whose
    host buffer cannot carry the lag still streams whenever it can; profiles/r02_ladder_study: C4 94.4 vs 92.1 GB/s
    drained, C5 equal); lag 0 -> the largest k <= max_lag that fits (1 if none)."""
    def fits(k):
        return host_free >= 1.1 * (1 + k) * off_max and free >= 1.1 * (up_max + (1 + k) * off_max)
    if retire == "auto":
        retire = "each"
    lag = retire_lag or max([k for k in range(1, max_lag + 1) if fits(k)] or [1])
    return retire, lag


# ------------------------------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import paper_2510_18586_b200 as tcb

    rank, world, local = dist_env()
    # TC_BENCH_DEVICE / TC_BENCH_BACKEND=gloo: rehearse the N-rank flow with every rank on one GPU (a box with a
    # single GPU cannot run NCCL between ranks sharing it); the timing numbers of such a run are not a scaling result
    local = int(os.environ.get("TC_BENCH_DEVICE", local))
    backend = os.environ.get("TC_BENCH_BACKEND", "nccl")
    numa = bind_numa_local(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    # TC_BENCH_DIST=1 (under torchrun): join the process group even at world size 1, so the N-rank code path — NCCL
    # barrier, all_reduce and all_gather of device tensors — runs on a one-GPU box
    if world > 1 or os.environ.get("TC_BENCH_DIST") == "1":
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg, G, scaling = workload_for(args, world)
    shard_rank = shard_rank_for(args, rank, G)
    mode_d2h, mode_h2d = {"auto": (tcb.XFER_AUTO,) * 2, "direct": (tcb.XFER_DIRECT,) * 2,
                          "staged": (tcb.XFER_STAGED,) * 2, "copy": (tcb.XFER_COPY,) * 2,
                          "mixed": (tcb.XFER_DIRECT, tcb.XFER_STAGED),
                          "mixed_rev": (tcb.XFER_STAGED, tcb.XFER_DIRECT)}[args.mode]
    if args.host_frac > 0:
        cfg = cfg.scaled(cfg.N, host_slots=max(1, int(cfg.N * args.host_frac)))
    S = cfg.host_slots()
    if args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but {world} rank(s) in this launch; n_gpus reports {world}",
              file=sys.stderr)

    # host-link peaks: each rank alone (the others wait at a barrier), then all ranks at once — the concurrent one is
    # the per-GPU denominator at N > 1 (shared PCIe switches / root complexes / host DRAM)
    link_alone, link = (None, None) if args.quick else link_probe(torch, dev, dist, rank, world)
    peer_dev = ((local + 1) % torch.cuda.device_count()) if args.peer else -1
    pool = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, cfg.N, device=local, shard_rank=shard_rank, shard_world=G,
                    host_slots=S, max_agents=1024, max_blocks_per_agent=cfg.max_blocks_per_agent,
                    xfer_d2h=mode_d2h, xfer_h2d=mode_h2d, peer_device=peer_dev, peer_slots=S if args.peer else 0)
    pool.fill(cfg.seed)
    B = pool.block_bytes
    calibration = None
    if args.mode == "auto" and os.environ.get("TC_BENCH_CALIBRATE", "1") != "0":
        calibration = pool.calibrate(256 << 20)   # AUTO re-measured on this box

    # setup (untimed): quotas, agents, decode-like interleaved pre-fill — through the C ABI
    ops, agents, _ = setup_ops(cfg)
    for op in ops:
        k = op[0]
        if k == "reserve":
            pool.reserve(op[1], op[2])
        elif k == "agent_add":
            pool.agent_add(op[1], op[2])
        elif k == "alloc":
            pool.alloc(op[1], op[2])
        elif k == "agent_free":
            pool.agent_free(op[1])
        elif k == "sync":
            pool.sync()
    gen = CycleGen(cfg, agents, combined=True)
    handles, sizes = {}, {}

    drains = [0]                               # refused cycles retried after a tc_sync
    ladders = [0]                              # refused cycles retried after a tc_retire (then maybe the sync)
    refused = {"nohost": 0, "noblocks": 0}     # why (first refusal of each laddered cycle)
    lag = [1]

    def cycle(record=None, retire="sync", on_uploads=None):
        """One scheduling cycle through the public API (tc_cycle: uploads then offloads), then its retirement point:
        retire = "sync" (tc_sync: drain and retire everything) or "retire" (tc_retire: retire what was enqueued
        before the previous point); returns (blocks_up, blocks_off)."""
        nu = no = 0
        started = False
        for op in gen.next_cycle():
            if op[0] == "cycle":
                hs = np.array([handles.pop(a) for a in op[1]], dtype=np.uint64)
                uoff = np.zeros(len(hs) + 1, dtype=np.int64)
                uoff[1:] = np.cumsum([sizes.pop(int(h)) for h in hs])
                ags = np.array([a for a, _ in op[2]], dtype=np.int32)
                tabs = [pool.block_table_np(int(a)) for a in ags]
                tabs = [t[t >= 0] for t in tabs]
                ooff = np.zeros(len(tabs) + 1, dtype=np.int64)
                ooff[1:] = np.cumsum([len(t) for t in tabs])
                ids = np.ascontiguousarray(np.concatenate(tabs)) if tabs else np.zeros(1, np.int32)
                if record is not None:
                    record("start")                 # just before the tc_cycle call
                    started = True
                try:
                    _, out_h = pool.cycle_arrays(hs, uoff, ags, ooff, ids)
                except tcb.TcError as e:            # refused, nothing changed (host buffer / blocks held by the
                    if e.status not in (tcb.E_NOHOST, tcb.E_NOBLOCKS) or retire == "sync":   # undrained cycles):
                        raise                       # retire the previous cycle's transfers and retry, then drain
                    pool.retire(1)
                    ladders[0] += 1
                    refused["nohost" if e.status == tcb.E_NOHOST else "noblocks"] += 1
                    try:
                        _, out_h = pool.cycle_arrays(hs, uoff, ags, ooff, ids)
                    except tcb.TcError as e2:
                        if e2.status not in (tcb.E_NOHOST, tcb.E_NOBLOCKS):
                            raise
                        pool.sync()
                        drains[0] += 1
                        _, out_h = pool.cycle_arrays(hs, uoff, ags, ooff, ids)
                for a, h, t in zip(ags, out_h, tabs):
                    handles[int(a)] = int(h)
                    sizes[int(h)] = len(t)
                if on_uploads is not None:
                    on_uploads(hs)
                nu += int(uoff[-1])
                no += int(ooff[-1])
            elif op[0] == "sync":
                if record is not None:
                    if not started:                 # a cycle with nothing to move: a zero-length step
                        record("start")
                    record("end")
                if retire == "sync":
                    pool.sync()
                else:
                    pool.retire(lag[0])
        return nu, no

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    up_s, off_s = pool.streams()
    ups, offs_ = torch.cuda.ExternalStream(up_s, device=dev), torch.cuda.ExternalStream(off_s, device=dev)

    clocks = Clocks(local)                     # sampled from warm-up through the end of the timed region
    for _ in range(cfg.stall_cycles + 1):      # prime: get stalled agents to upload
        cycle()
    warm = [cycle() for _ in range(max(args.warmup, 3))]
    s = pool.stats()
    args.retire, lag[0] = choose_retire(args.retire, args.retire_lag, s["host_free"], s["free"],
                                        max(u for u, _ in warm), max(o for _, o in warm))
    # timed region: the kernels' own %globaltimer start/end plus CUDA events around each kernel launch on its own
    # stream (timing mode 3; the DMAs carry no events, so the copy-engine schedule is untouched)
    pool.timing(3)
    pool.timing(3)                             # reset accumulators
    launches0 = pool.stats()["kernel_launches"]
    memcpy0 = pool.stats()["memcpy_calls"]
    # the host loop is a serving engine's scheduler: no cyclic-GC pause inside it (a gen-2 collection over torch's
    # heap takes milliseconds and lets the copy queues run dry); TC_BENCH_GC=1 keeps the collector on
    gc_off = os.environ.get("TC_BENCH_GC") != "1"
    trace_timed = os.environ.get("TC_TRACE_TIMED")          # experiments: per-call trace over the timed region
    if trace_timed:
        pool.trace(200000)
    if gc_off:
        gc.collect()
        gc.disable()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    dev_ms, host_ms, bytes_up, bytes_off, blocks, step_bytes = [], [], 0, 0, 0, []
    host_step_s = []                           # retire-each: host time per step (enqueue + the retire wait)
    t_wall0 = time.perf_counter()
    if args.retire == "each":
        # the asynchronous loop: each step enqueues its cycle and retires the previous one's transfers
        # (tc_retire) without draining its own, so consecutive cycles stream back to back; the last cycle is drained
        # by a tc_sync inside the timed region.  Device time = first step's start -> last step's end on both copy
        # streams.  No L2 flush: each step streams ~2x the 126 MB L2 through blocks the previous steps did not touch.
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for e, st in zip(e0, (ups, offs_)):
            e.record(st)
        drains[0] = ladders[0] = 0
        refused["nohost"] = refused["noblocks"] = 0
        for k in range(args.steps):
            th = time.perf_counter()
            nu, no = cycle(retire="retire")
            host_step_s.append(time.perf_counter() - th)
            step_bytes.append((nu * B, no * B))
            bytes_up += nu * B
            bytes_off += no * B
            blocks += nu + no
        for e, st in zip(e1, (ups, offs_)):
            e.record(st)
        pool.sync()
        torch.cuda.synchronize(dev)
        total_ms = max(e0[a].elapsed_time(e1[b]) for a in range(2) for b in range(2))
        dev_ms = [total_ms / args.steps] * args.steps
        host_ms = [(time.perf_counter() - t_wall0) * 1e3 / args.steps] * args.steps
    for _ in range(args.steps if args.retire == "sync" else 0):
        flush.zero_()                          # flush L2 between steps (outside the step's events)
        torch.cuda.synchronize(dev)
        ev = {}

        def record(tag):
            # device clock: from just before the tc_cycle call to the end of both copy streams' work
            pair = (("up0", ups), ("off0", offs_)) if tag == "start" else (("up1", ups), ("off1", offs_))
            for nm, st in pair:
                e = torch.cuda.Event(enable_timing=True); e.record(st); ev[nm] = e
        t0 = time.perf_counter()                # host clock (e2e): the whole public-API cycle incl. id lookups
        nu, no = cycle(record, retire="sync")
        t1 = time.perf_counter()
        ref = ev["up0"]
        start = min(0.0, ref.elapsed_time(ev["off0"]))
        end = max(ref.elapsed_time(ev["up1"]), ref.elapsed_time(ev["off1"]))
        dev_ms.append(end - start)
        host_ms.append((t1 - t0) * 1e3)
        step_bytes.append((nu * B, no * B))
        bytes_up += nu * B
        bytes_off += no * B
        blocks += nu + no
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    if gc_off:
        gc.enable()
    if trace_timed:
        with open(trace_timed, "w") as f:
            for r in pool.trace_read(200000):
                f.write(json.dumps(r) + "\n")
        pool.trace(0)
    clk = clocks.stop()
    tim = pool.timing(0)
    launches = pool.stats()["kernel_launches"] - launches0
    memcpys = pool.stats()["memcpy_calls"] - memcpy0     # DMA calls of the timed region only
    # diagnostic pass after the timed region (not in `value`): CUDA-event spans around every launch and DMA run, for
    # the per-direction DMA rates and the per-step timeline (events cost ~2 % of the step, so they stay out of it)
    pool.timing(1)
    pool.timing(1)
    pool.timeline_arm(200000)
    n_diag = min(args.steps, int(os.environ.get("TC_DIAG_STEPS", 20)))
    # TC_DIAG_RETIRE=1: run the diagnostic cycles in the timed loop's retire-each form (one timeline over all of
    # them, for TC_DUMP_TIMELINE / tools/timeline_gaps.py) instead of drained
    diag_each = args.retire == "each" and os.environ.get("TC_DIAG_RETIRE") == "1"
    # per-call records (host enqueue cost of rows a2 / a5, and --trace): each record's completion stamp is a host
    # callback queued on the copy stream, which holds the stream's next DMA until the host runs it — so not in a
    # retire-each timeline (it would show gaps the timed loop does not have)
    pool.trace(0 if diag_each else 100000)
    for _ in range(n_diag):
        cycle(retire="retire" if diag_each else "sync")
    if diag_each:
        pool.sync()
    trace_recs = pool.trace_read(100000)
    pool.trace(0)
    if args.trace and rank == 0:
        with open(args.trace, "w") as f:
            for r in trace_recs:
                f.write(json.dumps(r) + "\n")
    diag = pool.timing(0)
    tl_raw = pool.timeline(200000)
    other = per_cycle_drain(torch, dev, cycle, ups, offs_, B, min(args.steps, 40), flush, link) if args.retire == "each" \
        else None
    tl_summary = timeline_summary(tl_raw)
    if os.environ.get("TC_DUMP_TIMELINE"):                 # debugging aid: raw per-span records of the diagnostic steps
        with open(os.environ["TC_DUMP_TIMELINE"], "w") as f:
            json.dump(tl_raw, f)

    # the link re-measured after the timed region (all ranks at once, best of 3): a box whose link drifts shows it
    # here, next to the pre-loop best-of-10 peak that is the denominator of roofline_link
    link_after = None if (args.quick or not link) else hostlink_peak(torch, dev, reps=3)
    resume = None if args.quick else resume_probe(torch, dev, pool, cycle, ups, cfg.per_cycle)
    sweep = None
    if cfg.name == "c5" and not args.no_sweep:      # BASELINE configs[4]: 1-512 blocks per offload (every rank)
        if dist is not None:
            dist.barrier()
        sweep = offload_size_sweep(pool, cfg, B)
    my = torch.tensor([sum(dev_ms), sum(host_ms), bytes_up + bytes_off, blocks, t_wall,
                       link["bidir_gbs"] if link else 0.0], dtype=torch.float64,
                      device=dev if backend == "nccl" else "cpu")
    tot = my.clone()
    rows = [my.cpu().tolist()]
    if dist is not None:
        mx = my.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = my.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        tot = torch.stack([mx[0], mx[1], sm[2], sm[3], mx[4]])
        got = [torch.empty_like(my) for _ in range(world)]   # per-rank rows: flatness per GPU (the metric's "per GPU")
        dist.all_gather(got, my)
        rows = [g.cpu().tolist() for g in got]
    dev_total_ms, host_total_ms, all_bytes, all_blocks, wall = [float(x) for x in tot.cpu()[:5]]

    hbm, hbm_src = hbm_peak()
    dev_bench = None if args.quick else device_tier_bench(torch, pool, cfg, dev, hbm, hbm_src)
    if rank != 0:
        if dist is not None:
            dist.barrier(); dist.destroy_process_group()
        return

    value = all_bytes / (dev_total_ms * 1e-3) / 1e9
    e2e = all_bytes / (host_total_ms * 1e-3) / 1e9
    # roofline of the dominant kernel: per-launch algorithmic bytes / the launch's device duration
    stats = pool.stats()
    link_bound = {"offload_kernel": False, "upload_kernel": False, "offload_peer_kernel": False,
                  "upload_peer_kernel": False, "offload_direct_kernel": True, "upload_direct_kernel": True}
    kern = {}
    self_peer = args.peer and peer_dev == local
    for k, peak_key in (("offload_kernel", None), ("upload_kernel", None), ("offload_peer_kernel", None),
                        ("upload_peer_kernel", None), ("offload_direct_kernel", "d2h_gbs"),
                        ("upload_direct_kernel", "h2d_gbs")):
        # kernel duration = first CTA start -> last CTA end on the device clock (%globaltimer), recorded by the
        # kernel itself on the stream it runs on; the CUDA-event span around the launch (which also counts host
        # launch latency when the stream was idle) is kept beside it
        ms, cnt, byt = tim["dev_" + k]
        if not cnt:
            continue
        e = {"ms_total": ms, "launches": cnt, "bytes_per_launch": byt / cnt, "ms_per_launch": ms / cnt,
             "timing": "kernel-recorded %globaltimer first-CTA start -> last-CTA end, every launch of the timed region"}
        if "peer" in k and not self_peer:   # neighbour's HBM over NVLink: B per block over the link
            e.update(bound="nvlink", achieved=byt / (ms * 1e-3) / 1e9, peak=NVLINK_GBS,
                     peak_source="B200_PROFILING.md measured peer copy, per direction (900 nominal)")
        elif "peer" in k or not link_bound[k]:   # device-side kernel (staged, or a same-GPU peer slab): HBM r+w
            e.update(bound="hbm", achieved=2 * byt / (ms * 1e-3) / 1e9, peak=hbm, peak_source=hbm_src,
                     bytes_per_launch=2 * byt / cnt)
        else:                  # mapped-host kernel: every byte crosses the host link once
            pk = link[peak_key] if link else None
            e.update(bound="host_link", achieved=byt / (ms * 1e-3) / 1e9, peak=pk,
                     peak_source="live pinned cudaMemcpyAsync 1 GiB in this run (" + peak_key + ")")
            if link:
                e["frac_of_bidir_share"] = e["achieved"] / (link["bidir_gbs"] / 2)
        e["frac"] = e["achieved"] / e["peak"] if e["peak"] else None
        kern[k] = e
    for k in ("memcpy_d2h", "memcpy_h2d"):
        ms, cnt, byt = diag[k]
        if cnt:
            kern[k] = {"ms_total": ms, "runs": cnt, "achieved_gbs": byt / (ms * 1e-3) / 1e9,
                       "timing": f"CUDA-event spans around each DMA run, {n_diag} diagnostic steps after the timed region"}
    roof = None
    kern_only = {k: v for k, v in kern.items() if k.endswith("_kernel")}
    if kern_only:
        dom = max(kern_only, key=lambda k: kern_only[k]["ms_total"])
        kd = kern_only[dom]
        roof = {"kernel": dom, "bound": kd["bound"], "achieved": kd["achieved"], "peak": kd["peak"],
                "unit": "GB/s", "frac": kd["frac"], "traffic": None, "bytes_per_launch": kd["bytes_per_launch"],
                "ms_per_launch": kd["ms_per_launch"], "peak_source": kd["peak_source"],
                "share_of_kernel_time": kd["ms_total"] / sum(v["ms_total"] for v in kern_only.values())}
        if "peer" not in dom:
            roof.update(ncu_traffic(cfg.name, "gather" if dom.startswith("offload") else "scatter", kd))
        # the same kernel timed with CUDA events recorded on its own stream around every launch of the timed region
        # (timing mode 3): a launch whose stream was idle also counts its host-side launch latency
        ems, ecnt, ebytes = tim.get(dom, (0.0, 0, 0))
        if ecnt and ems:
            scale = 2 if kd["bound"] == "hbm" else 1           # HBM kernels count read + write, as above
            roof["event_check"] = {"ms_per_launch": ems / ecnt, "achieved": scale * ebytes / (ems * 1e-3) / 1e9,
                                   "frac": scale * ebytes / (ems * 1e-3) / 1e9 / kd["peak"] if kd["peak"] else None,
                                   "launches": ecnt, "how": "CUDA events on the kernel's own stream around every "
                                   "launch of the timed region (timing mode 3)"}
    # the step's binding resource is the host link: per-direction DMA/kernel rate and a per-step link roofline
    link_roof = None
    if link and not args.peer:
        bi = link["bidir_gbs"] / 2
        tmin = 0.0
        if args.retire == "each":              # steps stream back to back: the bound is on the totals
            up, off = sum(u for u, _ in step_bytes), sum(o for _, o in step_bytes)
            tmin = max(up / (link["h2d_gbs"] * 1e9), off / (link["d2h_gbs"] * 1e9), (up + off) / (link["bidir_gbs"] * 1e9))
            how = ("all steps: max(total up / H2D peak, total off / D2H peak, total / bidirectional peak), the link's "
                   "lower bound for any schedule, vs the measured time")
        else:
            tmin = sum(step_link_bound_s(u, o, link) for u, o in step_bytes)
            how = ("per step: min(up,off) at half the measured bidirectional peak + the excess at the unidirectional "
                   "peak, vs the measured step time")
        link_roof = {"bound": "host_link", "step_min_ms": tmin * 1e3 / len(step_bytes),
                     "step_ms": sum(dev_ms) / len(dev_ms), "frac": tmin * 1e3 / sum(dev_ms), "how": how}
        for k, pk in (("memcpy_d2h", "d2h_gbs"), ("memcpy_h2d", "h2d_gbs")):
            if k in kern:
                link_roof[k + "_frac_of_unidir_peak"] = kern[k]["achieved_gbs"] / link[pk]
                link_roof[k + "_frac_of_bidir_share"] = kern[k]["achieved_gbs"] / bi
    if self_peer and kern_only:
        # same-GPU peer slab: the offload and upload kernels read and write the same HBM at once, so each kernel's own
        # duration shows it sharing the bandwidth; the step's bound is HBM for both directions together
        hbm_bytes = 2 * all_bytes / world                    # every moved byte is read once and written once
        roof_step = {"bound": "hbm", "achieved": hbm_bytes / (dev_total_ms * 1e-3) / 1e9, "peak": hbm,
                     "peak_source": hbm_src, "how": "both directions' HBM read + write bytes / the timed region's "
                     "device time (the two peer kernels overlap and share HBM)"}
        roof_step["frac"] = roof_step["achieved"] / hbm if hbm else None
        roof["step_hbm"] = roof_step
    cpu = None
    if not args.no_cpu_baseline:               # rank 0, after the timed region (the other ranks wait at the barrier)
        cpu = cpu_baseline(cfg, args.cpu_seconds, G)
    n_steps = args.steps
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": n_steps, "warmup": args.warmup,
        "ms_per_step": dev_total_ms / n_steps, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "u16 (bit copy of bf16 KV)", "data": "synthetic (splitmix64 KV contents, seeded op scripts)",
        "config": {"workload": f"{cfg.name}: {cfg.title}", "layers": cfg.L, "kv_heads": cfg.H, "head_dim": cfg.D,
                   "block_tokens": cfg.T, "head_shards": G, "n_blocks": cfg.N, "block_shard_bytes": B,
                   "host_slots": S, "agents": cfg.n_agents, "per_cycle": cfg.per_cycle,
                   "xfer": XFER_NAMES[stats["xfer_d2h"]] + "/" + XFER_NAMES[stats["xfer_h2d"]],
                   "l2": ("not flushed: every step streams ~2x the 126 MB L2 through blocks the previous steps did "
                          "not touch" if args.retire == "each" else
                          "flushed between steps (256 MiB write, outside the step events)"),
                   "retire_lag": lag[0] if args.retire == "each" else None,
                   "ladder_refusals": dict(refused) if args.retire == "each" else None,
                   "step": (f"tc_cycle + tc_retire_lag({lag[0]}) (retire the transfers enqueued before the "
                            f"{lag[0]}-th previous point, do not drain the last {lag[0]} cycles'); "
                            "a cycle the host buffer / free blocks refuse is retried after a tc_retire, then once "
                            f"more after a tc_sync ({ladders[0]} of {n_steps} steps needed the retire, {drains[0]} the "
                            "sync); a tc_sync drains the last cycle inside the timed region" if args.retire == "each" else
                            "tc_cycle + tc_sync (drain and retire every cycle)"),
                   "parallelism": (f"one GPU running rank {shard_rank}'s shard of a {G}-GPU head-sharded run "
                                   "(its own host link; the per-GPU work of that run)" if args.head_shards else
                                   f"{world} independent ranks" + (f", head-sharded G={G}" if G > 1 else "")),
                   "shard_rank": shard_rank,
                   "numa": numa,
                   "offload_tier": ("peer slots on GPU %d (%s) first, then host" % (
                       peer_dev, "this GPU's own HBM" if peer_dev == local else "NVLink neighbour")) if args.peer
                   else "host"},
        "blocks_per_s": all_blocks / (dev_total_ms * 1e-3),
        "per_gpu": per_gpu_summary(rows),
        "bytes_per_step": all_bytes / n_steps,
        "gpu_launches": int(launches),
        "memcpy_calls_per_step": memcpys / n_steps,
        "kernels": kern,
        "auto_calibration": calibration,
        "sm_time_share": {
            "value": sum(v["ms_total"] for k, v in kern.items() if k.endswith("_kernel")) / sum(dev_ms),
            "how": "sum of the transfer kernels' device durations / the steps' device time: the fraction of the step "
                   "during which this path occupies SMs (the copy-engine DMAs use none); rank 0"},
        "timeline": tl_summary,
        "host_enqueue": host_enqueue_summary(trace_recs, dev_total_ms / n_steps),
        "host_steps": ({"p50_ms": statistics.median(host_step_s) * 1e3, "max_ms": max(host_step_s) * 1e3,
                        "first_ms": host_step_s[0] * 1e3,
                        "how": "retire-each: host wall time per step of the timed loop (tc_cycle + the retire wait); a "
                               "max far above p50 is a host-side stall"} if host_step_s else None),
        "per_cycle_drain": other,
        "hostlink_peak": link,
        "hostlink_peak_alone": link_alone,
        "hostlink_peak_after": link_after,
        "resume": resume,
        "sweep": sweep,
        "roofline": roof,
        "roofline_link": link_roof,
        "roofline_device": dev_bench,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": (bytes_up + 16 * all_blocks) / n_steps,
                "d2h_bytes_per_step": bytes_off / n_steps,
                "how": "host wall clock around the public-API loop (tc_cycle from host id arrays — uploads, then "
                       "offloads — and its retirement point, " + (f"tc_retire_lag({lag[0]}), a final tc_sync"
                       if args.retire == "each" else "tc_sync") + "), KV bytes crossing the host link inside it"},
        "cpu_baseline": cpu,
        "clocks": clk,
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier(); dist.destroy_process_group()


def ncu_traffic(cfg_name, kind, kd):
    """roofline.traffic for the staged HBM kernels: DRAM bytes per launch from the committed `ncu --set full` capture
    of fixed-size launches of the same kernel on the same config (tools/traffic_probe.py -> profiles/
    r<round>_traffic_<cfg>.json, the latest round's), as the captured ratio (dram read + write) / algorithmic bytes times this run's per-launch
    algorithmic bytes.  None when no capture exists or the kernel is a host-link one."""
    caps = [os.path.join(ROOT, "profiles", f"r{r:02d}_traffic_{cfg_name}.json") for r in (2, 1)]
    caps = [c for c in caps if os.path.exists(c)]                 # the latest round's capture first
    if kd.get("bound") != "hbm" or not caps:
        return {}
    path = caps[0]
    cap = [x for x in json.load(open(path))["launches"] if x["kind"] == kind]
    if not cap:
        return {}
    ratio = statistics.mean(x["ratio"] for x in cap)
    return {"traffic": ratio * kd["bytes_per_launch"],
            "traffic_source": {"capture": os.path.relpath(path, ROOT), "dram_over_algorithmic": ratio,
                               "dram_read_over_algorithmic_read": statistics.mean(x["read_ratio"] for x in cap),
                               "note": "ncu counts writes still dirty in L2 at kernel end as not yet written"}}


def step_link_bound_s(up: float, off: float, link: dict) -> float:
    """The host link's lower bound (s) for one drained step moving `up` bytes H2D and `off` bytes D2H: the smaller
    direction at half the measured bidirectional peak, the excess at the unidirectional peak of the larger one."""
    lo, hi = min(up, off), max(up, off)
    uni = link["h2d_gbs"] if up >= off else link["d2h_gbs"]
    return lo / (link["bidir_gbs"] / 2 * 1e9) + (hi - lo) / (uni * 1e9)


def per_cycle_drain(torch, dev, cycle, ups, offs, B, n, flush, link=None):
    """Diagnostic (not `value`): the same cycles run with a tc_sync each (drain and retire every cycle, L2 flushed
    between them); device time per cycle from just before tc_cycle to the end of both copy streams' work, and its
    fraction of the per-step link bound (a drained cycle pays its own up/off imbalance, which the bound includes)."""
    tot_ms, moved, bound_s = 0.0, 0, 0.0
    for _ in range(n):
        flush.zero_()
        torch.cuda.synchronize(dev)
        ev = {}

        def record(tag):
            for nm, st in ((tag + "u", ups), (tag + "o", offs)):
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                ev[nm] = e
        nu, no = cycle(record, retire="sync")
        if "startu" not in ev:
            continue
        tot_ms += max(ev["startu"].elapsed_time(ev["endu"]), ev["startu"].elapsed_time(ev["endo"]),
                      ev["starto"].elapsed_time(ev["endu"]), ev["starto"].elapsed_time(ev["endo"]))
        moved += (nu + no) * B
        if link:
            bound_s += step_link_bound_s(nu * B, no * B, link)
    return {"value": moved / (tot_ms * 1e-3) / 1e9 if tot_ms else None, "unit": "GB/s", "cycles": n,
            "link_frac": bound_s * 1e3 / tot_ms if (link and tot_ms) else None,
            "how": "tc_cycle + tc_sync per cycle (drained), L2 flushed between cycles; link_frac = sum of the "
                   "per-step link bounds / the measured time"}


def host_enqueue_summary(recs, step_ms):
    """Host cost of the integer rows of the path (a2 offload admission + host-slot pops + descriptors, a5 upload
    allocation, the table rewrite, the launches / DMA enqueues) per tc_cycle call, from the per-call trace: entry of
    the call -> the last of its batches enqueued.  Compared with the step's device time: the paper's pathology was
    exactly here."""
    cyc = {}
    for r in recs:
        c = cyc.setdefault(r["t_call_ns"], [0, 0])
        c[0] = max(c[0], r["t_enqueued_ns"] - r["t_call_ns"])
        c[1] += r["blocks"]
    if not cyc:
        return None
    us = sorted(v[0] / 1e3 for v in cyc.values())
    blocks = sum(v[1] for v in cyc.values())
    return {"cycles": len(us), "p50_us": us[len(us) // 2], "p99_us": us[min(len(us) - 1, int(0.99 * len(us)))],
            "mean_us": sum(us) / len(us), "ns_per_block": sum(us) * 1e3 / max(blocks, 1),
            "share_of_step": (sum(us) / len(us)) / (step_ms * 1e3) if step_ms else None,
            "how": "per tc_cycle: host ns from the call's entry to its last batch enqueued (tc_trace), diagnostic "
                   "steps; share = mean / the timed region's ms_per_step"}


def timeline_summary(spans):
    """Per sync interval (= step): when each kind of span first starts and last ends, relative to the step's first
    span; averaged over steps.  Shows how early each host-link direction starts and where the step's tail is."""
    by = {}
    for sync, kind, t0, t1, _ in spans:
        d = by.setdefault(sync, {})
        a, b = d.get(kind, (t0, t1))
        d[kind] = (min(a, t0), max(b, t1))
    if not by:
        return None
    kinds = sorted({k for d in by.values() for k in d})
    out = {}
    for k in kinds:
        v = [d[k] for d in by.values() if k in d]
        out[k] = {"first_start_ms": statistics.mean(x[0] for x in v), "last_end_ms": statistics.mean(x[1] for x in v)}
    out["step_span_ms"] = statistics.mean(max(x[1] for x in d.values()) for d in by.values())
    # per step: how late each DMA direction starts, and how long the step runs past its last DMA byte
    dma = [d for d in by.values() if "memcpy_d2h" in d and "memcpy_h2d" in d]
    if dma:
        out["d2h_start_ms"] = statistics.mean(d["memcpy_d2h"][0] for d in dma)
        out["h2d_start_ms"] = statistics.mean(d["memcpy_h2d"][0] for d in dma)
        out["tail_after_last_dma_ms"] = statistics.mean(
            max(x[1] for x in d.values()) - max(d["memcpy_d2h"][1], d["memcpy_h2d"][1]) for d in dma)
    out["steps"] = len(by)
    return out


def device_tier_bench(torch, pool, cfg, dev, hbm, hbm_src):
    """Device-side gather (KG1) and scatter (KS1) alone, >= 256 MiB per launch, event-timed (HBM roofline)."""
    B = pool.block_bytes
    n = max(1, (512 << 20) // B)
    rng = np.random.default_rng(7)
    ids = rng.choice(cfg.N, size=n, replace=False).astype(np.int32)
    dst = torch.empty(n * B, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    out = {}
    for name, fn in (("gather", lambda: pool.gather_dev(ids, dst.data_ptr(), s.cuda_stream)),
                     ("scatter", lambda: pool.scatter_dev(dst.data_ptr(), ids, s.cuda_stream))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        pool.sync()
        pool.timing(True)
        pool.timing(True)
        ts, dts = [], []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); fn(); e1.record(s); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
            pool.sync()                        # collects the kernel's own %globaltimer start/end
            dms, dcnt, _ = pool.timing(True)["dev_device_kernel"]
            if dcnt:
                dts.append(dms / dcnt)
        pool.timing(False)
        ms = statistics.median(dts) if dts else statistics.median(ts)
        ach = 2 * n * B / (ms * 1e-3) / 1e9
        out[name] = {"bytes_per_launch": n * B, "ms": ms, "achieved": ach, "frac": ach / hbm,
                     "event_ms_incl_launch": statistics.median(ts),
                     "how": "median of 10 launches; kernel-recorded %globaltimer first-CTA start -> last-CTA end"}
    return {"bound": "hbm", "unit": "GB/s (read+write)", "peak": hbm, "peak_source": hbm_src, **out,
            "note": "the kernel's end stamp does not wait for dirty L2 lines (126 MB L2) to reach DRAM, so a 512 MiB "
                    "launch can read up to ~6 % above the copy peak; DRAM reads/algorithmic reads = 1.0002 (ncu)"}


# ------------------------------------------------------------------------------------------------- CPU oracle
def oracle_scaled(cfg, G: int = 1):
    """The bounded host sample of a workload for the oracle: the rank's block shard (G head shards, so the same
    bytes per block as the GPU rank moves), a host-scaled pool of at most ~1.5 GB, at most 2 offloads + 2 uploads per
    cycle and (per_cycle x (stall_cycles + 2)) agents whose log-normal sizes are clamped so they all fit."""
    B = cfg.block_bytes(G)
    N = int(min(4096, max(256, (3 << 29) // B)))
    pc = min(cfg.per_cycle, 2)
    n_agents = pc * (cfg.stall_cycles + 2)
    hi = max(1, min(cfg.clamp[1], int(0.6 * N) // n_agents))
    lo = min(cfg.clamp[0], hi)
    return cfg.scaled(N=N, host_slots=int(N * 0.45), bg_fill=0.2, per_cycle=pc, n_agents=n_agents,
                      med_blocks=min(cfg.med_blocks, hi), clamp=(lo, hi), G=G, churn=0.0)


def oracle_setup(cfg, G: int = 1):
    """The oracle (BytesStore: real pool and host-slot arrays) set up on oracle_scaled(cfg, G)."""
    from oracle import BytesStore, OraclePool
    small = oracle_scaled(cfg, G)
    N = small.N
    C = small.chunk_bytes(G)
    pool0 = np.empty((small.L, 2, N, C), dtype=np.uint8)
    pool0.fill(0xA5)                                   # content is irrelevant to the timing of byte copies
    o = OraclePool(N, small.host_slots(), max_agents=1024, max_blocks_per_agent=small.max_blocks_per_agent,
                   store=BytesStore(pool0, small.host_slots()))
    from workloads.replay import Replayer
    ops, agents, _ = setup_ops(small)
    tr = Replayer(o).run(ops)
    assert all(st == 0 for st, _ in tr), "host sample does not fit its pool"
    return small, o, agents


def oracle_cycles(small, o, agents, seconds=None, steps=None, warmup=0):
    from workloads.replay import Replayer
    gen = CycleGen(small, agents)
    r = Replayer(o)
    for a in agents:
        r.handles.setdefault(a, __import__("collections").deque())
    B = small.block_bytes(small.G)

    def one():
        nb = 0
        for op in gen.next_cycle():
            st, out = r.step(op)
            assert st == 0, op
            if op[0] == "upload_batch":
                nb += sum(len(x) for x in out)
            elif op[0] == "offload_batch":
                nb += sum(r.pool.handles[h].pos.__len__() for h in out)
        return nb

    for _ in range(small.stall_cycles + 1 + warmup):
        one()
    t0 = time.perf_counter()
    times, blocks = [], 0
    while True:
        s = time.perf_counter()
        blocks += one()
        times.append(time.perf_counter() - s)
        if steps is not None and len(times) >= steps:
            break
        if seconds is not None and time.perf_counter() - t0 >= seconds:
            break
    return blocks * B, sum(times), len(times)


def cpu_baseline(cfg, seconds, G: int = 1):
    small, o, agents = oracle_setup(cfg, G)
    nbytes, secs, cycles = oracle_cycles(small, o, agents, seconds=seconds)
    return {"value": nbytes / secs / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{cycles} cycles of {cfg.name} ({small.per_cycle} offloads + uploads per cycle, "
                      f"{small.n_agents} agents, log-normal sizes clamped to [{small.clamp[0]}, {small.clamp[1]}] "
                      f"blocks) on a host-scaled pool (N={small.N}, {small.host_slots()} slots, "
                      f"{small.block_bytes(G)}-byte block shards, G={G}), NumPy BytesStore, single thread, "
                      f"{secs:.1f} s",
            "host_cpu_count": os.cpu_count()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, G, scaling = workload_for(args, world)
    small, o, agents = oracle_setup(cfg, G)
    nbytes, secs, cycles = oracle_cycles(small, o, agents, steps=args.steps, warmup=args.warmup)
    value = nbytes / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / cycles, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u16 (bit copy of bf16 KV)", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.title}", "host_scaled_n_blocks": small.N, "head_shards": G,
                   "block_shard_bytes": small.block_bytes(G)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{cycles} cycles of {cfg.name} ({small.per_cycle} offloads + uploads per cycle, "
                                   f"{small.n_agents} agents, sizes clamped to [{small.clamp[0]}, {small.clamp[1]}]) "
                                   f"on a host-scaled pool (N={small.N}, {small.block_bytes(G)}-byte block shards)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_dry(args):
    """--dry-run: the N-rank plumbing without a GPU — rendezvous (gloo), the workload each rank would run, the
    per-rank rows gathered to rank 0, the barrier / max / sum reductions, and rank 0's cpu_baseline."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    cfg, G, scaling = workload_for(args, world)
    shard_rank = shard_rank_for(args, rank, G)
    my = torch.tensor([1.0, 1.0, float(cfg.block_bytes(G)), 1.0, 0.0, 0.0], dtype=torch.float64)
    rows = [my.tolist()]
    shards = [shard_rank]
    if world > 1:
        dist.barrier()
        got = [torch.empty_like(my) for _ in range(world)]
        dist.all_gather(got, my)
        rows = [g.tolist() for g in got]
        sr = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sr, torch.tensor([shard_rank], dtype=torch.int64))
        shards = [int(x) for x in sr]
    cpu = cpu_baseline(cfg, args.cpu_seconds, G) if rank == 0 and not args.no_cpu_baseline else None
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "scaling": scaling,
                          "config": {"workload": f"{cfg.name}: {cfg.title}", "head_shards": G,
                                     "shard_ranks": shards, "block_shard_bytes": cfg.block_bytes(G),
                                     "parallelism": f"{world} ranks" + (f", head-sharded G={G}" if G > 1 else "")},
                          "per_gpu": per_gpu_summary(rows), "cpu_baseline": cpu}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    rc = self_launch(a, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    if a.dry_run:
        run_dry(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
