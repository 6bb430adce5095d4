"""Transfer-path tuning probe (GPU box): per-launch kernel GB/s of the direct D2H / H2D kernels (SIMT vs TMA bulk,
CTA counts), alone and concurrent, vs the staged copy-engine path.  Prints one JSON object per configuration and
writes gpurun_out/xfer_probe.json.  Tuning aid only; the bench is bench.py."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T = int(os.environ.get("PL", 28)), int(os.environ.get("PH", 4)), 128, 16
N, S, NB = 8192, 2048, int(os.environ.get("PNB", 256))
REPS = 5


def main():
    p = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=S, max_blocks_per_agent=8192)
    p.fill(3)
    p.agent_add(0, 0); p.agent_add(1, 0); p.agent_add(2, 1)
    for _ in range(NB):
        p.alloc(0, 1); p.alloc(2, 1); p.alloc(1, 1); p.alloc(2, 1)
    B = p.block_bytes
    res = []

    def run(mode, path_cfg, concurrent):
        p.set_xfer_mode(mode, mode)
        for path, (ctas, thr, var) in path_cfg.items():
            p.set_launch_config(path, ctas, thr, var)
        out = []
        for rep in range(REPS + 1):
            p.timing(True)
            if concurrent:
                ha = p.offload(0, p.block_table(0)); p.sync()
                t0 = time.perf_counter()
                p.upload_batch([ha])
                hb = p.offload(1, p.block_table(1))
                p.sync()
                t1 = time.perf_counter()
                tim = p.timing(True)
                p.upload(hb); p.sync()
            else:
                t0 = time.perf_counter()
                h = p.offload(0, p.block_table(0)); p.sync()
                p.upload(h); p.sync()
                t1 = time.perf_counter()
                tim = p.timing(True)
            if rep:
                out.append((tim, t1 - t0))
        agg = {}
        for k in ("offload_kernel", "upload_kernel", "offload_direct_kernel", "upload_direct_kernel", "memcpy_d2h",
                  "memcpy_h2d"):
            ms = [t[k][0] for t, _ in out if t[k][1]]
            by = [t[k][2] for t, _ in out if t[k][1]]
            if ms:
                agg[k] = round(float(np.median([b / (m * 1e-3) / 1e9 for b, m in zip(by, ms)])), 2)
        return agg, float(np.median([w for _, w in out])) * 1e3

    cfgs = []
    grids = {0: (64, 148, 296, 592), 1: (32, 64, 148), 2: (148, 296, 592, 1184), 3: (64, 148, 296)}
    for var in (0, 1, 2, 3):
        for ctas in grids[var]:
            cfgs.append(("direct", var, ctas))
    cfgs.append(("staged", 0, 0))
    for conc in (False, True):
        for mode, var, ctas in cfgs:
            m = tcb.XFER_DIRECT if mode == "direct" else tcb.XFER_STAGED
            cfg = {0: (ctas, 256, var), 1: (ctas, 256, var), 2: (0, 256, 3)}
            try:
                agg, wall = run(m, cfg, conc)
            except tcb.TcError as e:
                agg, wall = {"error": str(e)}, None
                print(json.dumps({"mode": mode, "variant": var, "ctas": ctas, "concurrent": conc, **agg}), flush=True)
                return res
            r = {"mode": mode, "variant": var, "ctas": ctas, "concurrent": conc, "blocks": NB,
                 "mib": NB * B / 2**20, "wall_ms": wall, **agg}
            res.append(r)
            print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/xfer_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    main()
