"""Device-side gather/scatter tuning probe (GPU box): kernel-recorded duration (%globaltimer) of the device tier
(KG1/KS1) per variant x grid x launch size, on a C2-shaped pool (or PL/PH env), against the measured HBM copy peak.
Tuning aid only; the bench is bench.py.  Writes gpurun_out/tier_probe.json."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

L, H, D, T = int(os.environ.get("PL", 28)), int(os.environ.get("PH", 4)), 128, 16
N = int(os.environ.get("PN", 16384))
REPS = 10


def main():
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    p = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=16)
    p.fill(3)
    B = p.block_bytes
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rng = np.random.default_rng(7)
    sizes_mib = [int(x) for x in os.environ.get("PSIZES", "1,4,32,104,512").split(",")]
    variants = [int(x) for x in os.environ.get("PVARS", "0,1,2,3").split(",")]
    grids = {0: [0], 1: [0, 296], 2: [0, 1184, 2368], 3: [0, 444, 592]}
    if os.environ.get("PGRIDS"):
        grids = json.loads(os.environ["PGRIDS"])
        grids = {int(k): v for k, v in grids.items()}
    dst = torch.empty((max(sizes_mib) << 20) + B, dtype=torch.uint8, device=dev)
    res = []
    for mib in sizes_mib:
        n = max(1, (mib << 20) // B)
        ids = rng.choice(N, size=n, replace=False).astype(np.int32)
        for var in variants:
            for ctas in grids[var]:
                p.set_launch_config(2, ctas, 256, var)
                row = {"mib": round(n * B / 2**20, 1), "blocks": n, "variant": var, "ctas": ctas}
                for name, fn in (("gather", lambda: p.gather_dev(ids, dst.data_ptr(), s.cuda_stream)),
                                 ("scatter", lambda: p.scatter_dev(dst.data_ptr(), ids, s.cuda_stream))):
                    fn()
                    torch.cuda.synchronize(dev)
                    p.sync()
                    p.timing(True)
                    p.timing(True)
                    dts = []
                    for _ in range(REPS):
                        flush.zero_()
                        torch.cuda.synchronize(dev)
                        fn()
                        torch.cuda.synchronize(dev)
                        p.sync()
                        dms, dcnt, _ = p.timing(True)["dev_device_kernel"]
                        if dcnt:
                            dts.append(dms / dcnt)
                    p.timing(False)
                    ms = statistics.median(dts)
                    ach = 2 * n * B / (ms * 1e-3) / 1e9
                    row[name + "_us"] = round(ms * 1e3, 2)
                    row[name + "_frac"] = round(ach / peak, 3)
                res.append(row)
                print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/tier_probe.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
