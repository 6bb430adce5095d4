"""DIRECT-mode probe (GPU box): the mapped-host gather (D2H) and scatter (H2D) kernels running CONCURRENTLY, as one
tc_cycle moves them, per launch configuration (variant x CTAs x threads) — the question being why SM-driven
bidirectional traffic stalls far below the link's bidirectional copy-engine rate.  Per configuration: each
direction's kernel-stamped GB/s, the cycle's device time (events on both copy streams) and its combined GB/s, the
overlap of the two kernels (how much of the shorter one ran while the other was running).

  python tools/direct_probe.py [--blocks 256] [--geom c2|c5] [--quick]
Writes gpurun_out/direct_probe.json.  Tuning aid; the bench is bench.py.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

GEOMS = {"c2": (28, 4, 128, 1), "c5": (80, 8, 128, 8)}   # L, H, D, G


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=256)
    ap.add_argument("--geom", default="c2")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--focus", action="store_true",
                    help="candidate configs only: each direction alone and both together, and the mixed pairs "
                         "(direct D2H + staged H2D, staged D2H + direct H2D)")
    a = ap.parse_args()
    L, H, D, G = GEOMS[a.geom]
    NB = a.blocks
    N, S = 4 * NB + 64, 3 * NB + 16
    p = tcb.Pool(L, H, D, 16, "bf16", N, device=0, shard_world=G, host_slots=S, max_blocks_per_agent=4 * NB,
                 xfer_d2h=tcb.XFER_DIRECT, xfer_h2d=tcb.XFER_DIRECT)
    p.fill(3)
    p.agent_add(0, 0)
    p.agent_add(1, 0)
    p.agent_add(2, 1)
    for _ in range(NB):                       # scattered ids: three agents grown interleaved
        p.alloc(0, 1)
        p.alloc(2, 1)
        p.alloc(1, 1)
    p.sync()
    B = p.block_bytes
    up_s, off_s = p.streams()
    ups = torch.cuda.ExternalStream(up_s, device=0)
    offs = torch.cuda.ExternalStream(off_s, device=0)
    res = []

    def one(cfg, modes=(tcb.XFER_DIRECT, tcb.XFER_DIRECT), which="both"):
        p.set_xfer_mode(*modes)
        for path in (0, 1):
            p.set_launch_config(path, *cfg[path])
        h = p.offload(0, p.block_table(0))     # agent 0 on the host: its upload runs beside agent 1's offload
        p.sync()
        rows = []
        for rep in range(a.reps + 1):
            p.timing(2)
            p.timing(2)
            e0u, e0o = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e1u, e1o = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0u.record(ups)
            e0o.record(offs)
            _, hs = p.cycle([h] if which != "off" else [], [(1, p.block_table(1))] if which != "up" else [])
            e1u.record(ups)
            e1o.record(offs)
            p.sync()
            tim = p.timing(0)
            wall = max(e0u.elapsed_time(e1u), e0u.elapsed_time(e1o), e0o.elapsed_time(e1u), e0o.elapsed_time(e1o))
            off_ms, off_n, off_b = tim["dev_offload_direct_kernel"]
            up_ms, up_n, up_b = tim["dev_upload_direct_kernel"]
            moved = (NB * B if which != "up" else 0) + (NB * B if which != "off" else 0)
            if which != "up":
                p.upload(hs[0])                # agent 1 back on the GPU (the next rep offloads it again)
                p.sync()
            if which != "off":
                h = p.offload(0, p.block_table(0))
                p.sync()
            if rep:
                rows.append({"off_gbs": off_b / (off_ms * 1e-3) / 1e9 if off_ms else None,
                             "up_gbs": up_b / (up_ms * 1e-3) / 1e9 if up_ms else None,
                             "cycle_gbs": moved / (wall * 1e-3) / 1e9, "cycle_ms": wall,
                             "off_ms": off_ms or None, "up_ms": up_ms or None})
        p.upload(h)
        p.sync()
        med = {k: float(np.median([r[k] for r in rows if r[k] is not None])) for k in rows[0]
               if any(r[k] is not None for r in rows)}
        # overlap: if the kernels ran one after the other, cycle_ms ~ off_ms + up_ms; fully overlapped ~ max(..)
        if "off_ms" in med and "up_ms" in med:
            med["serial_fraction"] = (med["cycle_ms"] - max(med["off_ms"], med["up_ms"])) / min(med["off_ms"],
                                                                                               med["up_ms"])
        return med

    if a.focus:
        names = {tcb.XFER_DIRECT: "direct", tcb.XFER_STAGED: "staged"}
        cands = [(592, 128, 0), (296, 256, 0), (74, 256, 0), (74, 32, 3), (32, 32, 3), (16, 32, 3), (74, 32, 1),
                 (148, 32, 3), (74, 256, 4), (148, 256, 4), (296, 256, 4), (592, 128, 4)]
        if os.environ.get("DP_CANDS"):                # e.g. DP_CANDS="74,256,4;148,256,4"
            cands = [tuple(int(x) for x in c.split(",")) for c in os.environ["DP_CANDS"].split(";")]
        D, St = tcb.XFER_DIRECT, tcb.XFER_STAGED
        for cand in cands:
            cfg = {0: cand, 1: cand}
            for modes, which in (((D, D), "off"), ((D, D), "up"), ((D, D), "both"), ((D, St), "both"),
                                 ((St, D), "both")):
                med = one(cfg, modes, which)
                r = {"geom": a.geom, "blocks": NB, "cfg": list(cand), "d2h": names[modes[0]], "h2d": names[modes[1]],
                     "which": which, **{k: round(v, 3) for k, v in med.items()}}
                res.append(r)
                print(json.dumps(r), flush=True)
        med = one({0: cands[0], 1: cands[0]}, (St, St), "both")
        r = {"geom": a.geom, "blocks": NB, "d2h": "staged", "h2d": "staged", "which": "both",
             **{k: round(v, 3) for k, v in med.items()}}
        res.append(r)
        print(json.dumps(r), flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/direct_focus_{a.geom}.json", "w") as f:
            json.dump(res, f, indent=1)
        return

    grid_set = (16, 32, 74, 148, 296, 592) if not a.quick else (32, 148, 592)
    cfgs = []
    for var in (0, 2):
        for thr in (128, 256):
            for ctas in grid_set:
                cfgs.append({0: (ctas, thr, var), 1: (ctas, thr, var)})
    for var in (1, 3):
        for ctas in grid_set:
            cfgs.append({0: (ctas, 32, var), 1: (ctas, 32, var)})
    # asymmetric splits: the H2D (read) kernel gets more CTAs than the D2H (write) kernel and vice versa
    for c0, c1 in ((32, 148), (148, 32), (74, 296), (296, 74)):
        cfgs.append({0: (c0, 256, 0), 1: (c1, 256, 0)})
    for cfg in cfgs:
        try:
            med = one(cfg)
        except tcb.TcError as e:
            print(json.dumps({"cfg": str(cfg), "error": str(e)}), flush=True)
            continue
        r = {"geom": a.geom, "blocks": NB, "block_bytes": B, "d2h": list(cfg[0]), "h2d": list(cfg[1]),
             **{k: round(v, 3) for k, v in med.items()}}
        res.append(r)
        print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/direct_probe_{a.geom}.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
