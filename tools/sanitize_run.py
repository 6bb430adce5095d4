"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel
path of the library — fill, staged TMA gather/scatter (single piece, pieces, ring reuse), direct mapped-host kernels
of every variant, COPY mode's table kernel, the device tier and the peer tier — over small C1/C2-shaped pools.
Exercises only; parity is the -m gpu suite's job."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import c1_worked_example, fuzz_script  # noqa: E402

RUNS = [  # (name, L, H, D, N, S, d2h, h2d, variant, staging, peer)
    ("c1-auto", 1, 2, 64, 64, 16, tcb.XFER_AUTO, tcb.XFER_AUTO, None, 0, 0),
    ("c1-staged-ring", 1, 2, 64, 64, 16, tcb.XFER_STAGED, tcb.XFER_STAGED, 3, 3 * 8192, 0),
    ("c2ish-staged", 4, 4, 128, 40, 16, tcb.XFER_STAGED, tcb.XFER_STAGED, 3, 0, 0),
    ("c2ish-direct-v0", 4, 4, 128, 40, 16, tcb.XFER_DIRECT, tcb.XFER_DIRECT, 0, 0, 0),
    ("c2ish-direct-v1", 4, 4, 128, 40, 16, tcb.XFER_DIRECT, tcb.XFER_DIRECT, 1, 0, 0),
    ("c2ish-direct-v2", 4, 4, 128, 40, 16, tcb.XFER_DIRECT, tcb.XFER_DIRECT, 2, 0, 0),
    ("c2ish-direct-default", 4, 4, 128, 40, 16, tcb.XFER_DIRECT, tcb.XFER_DIRECT, None, 0, 0),
    ("c2ish-direct-v4", 4, 4, 128, 40, 16, tcb.XFER_DIRECT, tcb.XFER_DIRECT, 4, 0, 0),
    ("c2ish-staged-v4", 4, 4, 128, 40, 16, tcb.XFER_STAGED, tcb.XFER_STAGED, 4, 0, 0),
    ("c2ish-staged-2blocks", 4, 4, 128, 40, 16, tcb.XFER_STAGED, tcb.XFER_STAGED, None, 1, 0),
    ("c2ish-copy", 4, 4, 128, 40, 16, tcb.XFER_COPY, tcb.XFER_COPY, None, 0, 0),
    ("c2ish-peer", 4, 4, 128, 40, 16, tcb.XFER_STAGED, tcb.XFER_STAGED, None, 0, 8),
]


def main():
    force = os.environ.get("SAN_VARIANT")      # e.g. 2: SIMT kernels only (initcheck does not track TMA bulk stores)
    for name, L, H, D, N, S, d2h, h2d, var, staging, peer in RUNS:
        if force is not None:
            var = int(force)
        p = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, n_classes=2, xfer_d2h=d2h, xfer_h2d=h2d,
                     staging_bytes=staging, peer_device=0 if peer else -1, peer_slots=peer)
        if var is not None:
            for path in range(4):
                p.set_launch_config(path, 0, 256, var)
        p.fill(3)
        r = Replayer(p)
        ops = c1_worked_example() if name.startswith("c1") else []
        ops += fuzz_script(11, n_ops=60, n_agents=3, n_classes=2, N=N, max_alloc=6, gradual=True, retire=True,
                           lags=(1, 2, 3))
        tr = r.run(ops)
        p.sync()
        ids = np.arange(min(8, N), dtype=np.int32)
        buf = torch.empty(len(ids) * p.block_bytes, dtype=torch.uint8, device="cuda:0")
        p.gather_dev(ids, buf.data_ptr())
        p.scatter_dev(buf.data_ptr(), ids)
        torch.cuda.synchronize()
        p.close()
        print(name, "ok", sum(1 for s, _ in tr if s == 0), "of", len(tr), "ops succeeded", flush=True)


if __name__ == "__main__":
    main()
