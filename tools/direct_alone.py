"""One DIRECT offload (mapped-host writes) and one DIRECT upload (mapped-host reads) of 256 C2-shaped blocks
(235 MB each way) with the library's default DIRECT launch configuration (TMA bulk, 32 / 74 CTAs), one after the
other — the workload for an `ncu --set full` capture of the two DIRECT kernels alone (PCIe counters).
    ncu --set full -k regex:k_xfer_bulk -o gpurun_out/prof_direct_alone python tools/direct_alone.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_18586_b200 as tcb  # noqa: E402

NB = 256
p = tcb.Pool(28, 4, 128, 16, "bf16", 4 * NB, device=0, host_slots=2 * NB, xfer_d2h=tcb.XFER_DIRECT,
             xfer_h2d=tcb.XFER_DIRECT)
p.fill(3)
p.agent_add(0, 0)
p.agent_add(1, 0)
for _ in range(NB):                                   # scattered ids
    p.alloc(0, 1)
    p.alloc(1, 1)
p.sync()
h = p.offload(0, p.block_table(0))                    # DIRECT D2H kernel
p.sync()
p.upload(h)                                           # DIRECT H2D kernel
p.sync()
p.close()
print("direct alone ok")
