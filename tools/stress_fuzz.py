"""Long randomized GPU stress against the CPU oracle (GPU box): fuzz scripts (error paths, batches, cycles, gradual
reservation, retire lags) replayed on the oracle and on the library side by side, over every transfer mode and
several geometries with ragged chunk counts, with TC_CHECK=1 (SPEC invariants + launch-descriptor bounds after every
call).  After every sync: the whole device pool, every block table (host mirror and device table) and the counters;
after every successful offload: every live host image.  Runs until the time budget is spent; prints one JSON line
(ops, syncs compared, bytes compared, mismatches = 0 or the first failure).

    TC_CHECK=1 python tools/stress_fuzz.py [seconds=900]
Test infrastructure (imports oracle/).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from oracle import BytesStore, OraclePool  # noqa: E402
from oracle.pool import OFFLOADED  # noqa: E402
from workloads import content  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import fuzz_script  # noqa: E402

MODES = [(tcb.XFER_STAGED, tcb.XFER_STAGED, 3), (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 3), (tcb.XFER_AUTO, tcb.XFER_AUTO, 3),
         (tcb.XFER_DIRECT, tcb.XFER_STAGED, 2), (tcb.XFER_COPY, tcb.XFER_STAGED, 3), (tcb.XFER_STAGED, tcb.XFER_COPY, 0),
         (tcb.XFER_STAGED, tcb.XFER_STAGED, 4), (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 1)]
GEOMS = [(1, 2, 64, 64, 16, 16), (3, 2, 64, 50, 20, 16), (5, 4, 128, 40, 24, 16), (2, 8, 128, 33, 12, 16),
         (7, 1, 8, 29, 9, 3), (4, 4, 128, 96, 48, 16)]


def full_compare(o, c):
    kv = c.kv_tensor().cpu().numpy()
    if not np.array_equal(kv, o.store.pool):
        return "pool bytes", 0
    for a in o.agents:
        if o.block_table(a) != c.block_table(a):
            return f"block table {a}", kv.nbytes
    tab = c.table_tensor().cpu().numpy()
    for a, ag in o.agents.items():
        if tab[a, :len(ag.table)].tolist() != ag.table:
            return f"device table {a}", kv.nbytes
    so, sc = o.stats(), c.stats()
    for k in ("free", "alloc", "pending", "reserved_blocks", "host_free", "host_used", "reserved", "claimed"):
        if so[k] != sc[k]:
            return f"counter {k}", kv.nbytes
    return None, kv.nbytes


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 900.0
    t0 = time.time()
    ops_done = syncs = host_imgs = 0
    bytes_cmp = 0
    runs = 0
    failure = None
    seed = 0
    while time.time() - t0 < budget and failure is None:
        L, H, D, N, S, T = GEOMS[seed % len(GEOMS)]
        d2h, h2d, variant = MODES[(seed // len(GEOMS)) % len(MODES)]
        B = 2 * L * T * H * D * 2
        staging = [0, 3 * B, 5 * B][seed % 3]
        pool0 = content.pool_bytes(seed + 1, L, N, T, H, D)
        o = OraclePool(N, S, n_classes=2, max_agents=1024, store=BytesStore(pool0, S))
        c = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=S, n_classes=2, max_agents=1024,
                     xfer_d2h=d2h, xfer_h2d=h2d, staging_bytes=staging)
        for path in range(3):
            c.set_launch_config(path, 0, 256, variant)
        c.fill(seed + 1)
        ops = fuzz_script(50_000 + seed, n_ops=400, n_agents=4, n_classes=2, N=N, max_alloc=6,
                          gradual=seed % 2 == 0, retire=True, lags=(1, 2, 3))
        ro, rc = Replayer(o), Replayer(c)
        for i, op in enumerate(ops):
            a, b = ro.step(op), rc.step(op)
            ops_done += 1
            if a != b:
                failure = {"seed": seed, "op": i, "what": repr(op), "oracle": repr(a), "library": repr(b)}
                break
            if op[0] in ("offload", "offload_batch", "cycle") and a[0] == 0:
                for h, hd in o.handles.items():
                    if hd.state != OFFLOADED:
                        continue
                    c.wait(h)
                    for k, s in enumerate(hd.slots):
                        host_imgs += 1
                        if not np.array_equal(c.handle_host_bytes(h, k), o.store.host[s]):
                            failure = {"seed": seed, "op": i, "what": f"host image {h}/{k}"}
                            break
                    if failure:
                        break
            if failure:
                break
            if op[0] == "sync":
                what, nb = full_compare(o, c)
                syncs += 1
                bytes_cmp += nb
                if what:
                    failure = {"seed": seed, "op": i, "what": what}
                    break
        if failure is None:
            c.sync()
            o.sync()
            what, nb = full_compare(o, c)
            syncs += 1
            bytes_cmp += nb
            if what:
                failure = {"seed": seed, "op": "end", "what": what}
        c.close()
        runs += 1
        seed += 1
    print(json.dumps({"seconds": round(time.time() - t0, 1), "scripts": runs, "ops": ops_done,
                      "full_state_compares": syncs, "host_images_compared": host_imgs,
                      "pool_bytes_compared": bytes_cmp, "tc_check": os.environ.get("TC_CHECK") == "1",
                      "mismatches": 0 if failure is None else 1, "first_failure": failure}), flush=True)
    sys.exit(0 if failure is None else 1)


if __name__ == "__main__":
    main()
