#!/bin/bash
# Is the loop's H2D shortfall on some boxes a host-memory property?  The footprint probe with torch-pinned and
# library-style (Portable|Mapped) 16 GiB slabs, then the default C3 bench line (loop H2D vs the probe) on the same box.
V=${V:-v1}
mkdir -p gpurun_out
python tools/footprint_probe.py 16 6 64 torch > gpurun_out/fpbox_torch_$V.jsonl 2>&1
python tools/footprint_probe.py 16 6 64 lib > gpurun_out/fpbox_lib_$V.jsonl 2>&1
timeout 600 python3 bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fpbox_c3_$V.json 2> gpurun_out/fpbox_c3_$V.err
cat gpurun_out/fpbox_torch_$V.jsonl gpurun_out/fpbox_lib_$V.jsonl
python - <<PY
import json
d = json.loads(open("gpurun_out/fpbox_c3_$V.json").read().strip().splitlines()[-1])
k = d["kernels"]
print("c3", round(d["value"], 2), "probe split", d["hostlink_peak"].get("bidir_split_gbs"), "loop h2d", round(k["memcpy_h2d"]["achieved_gbs"], 1),
      "d2h", round(k["memcpy_d2h"]["achieved_gbs"], 1))
PY
