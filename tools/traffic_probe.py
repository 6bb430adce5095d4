"""Fixed-size device-side gather + scatter launches for an `ncu --set full` DRAM-traffic capture (GPU box):
  ncu --set full -k regex:k_xfer_bulk -o gpurun_out/prof_traffic python tools/traffic_probe.py [config [MiB]]
Each launch moves a known number of blocks, so its algorithmic bytes (2 x n x B: read + write) are exact; the
capture's dram__bytes_read/write per launch divided by them is the traffic ratio bench.py reports."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = CONFIGS[name]
    G = cfg.G if name == "c5" else 1
    N = 8192
    p = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, N, device=0, shard_world=G, host_slots=16)
    p.fill(3)
    B = p.block_bytes
    mib = int(sys.argv[2]) if len(sys.argv) > 2 else 112   # default ~ one C2 scheduling cycle's offload
    n = max(1, (mib << 20) // B)
    ids = np.random.default_rng(7).choice(N, size=n, replace=False).astype(np.int32)
    dst = torch.empty(n * B, dtype=torch.uint8, device="cuda:0")
    for _ in range(2):
        p.gather_dev(ids, dst.data_ptr())
        p.scatter_dev(dst.data_ptr(), ids)
    torch.cuda.synchronize()
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/traffic_probe_{name}.json", "w") as f:
        json.dump({"config": name, "blocks": int(n), "block_bytes": int(B), "algorithmic_bytes": int(2 * n * B),
                   "launch_order": ["gather", "scatter", "gather", "scatter"]}, f)
    print("blocks", n, "B", B)


if __name__ == "__main__":
    main()
