#!/bin/bash
# Run-to-run distribution of the driver's default command (C3) on one box: 8 back-to-back runs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3 4 5 6 7 8; do
  timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 $( [ $r -gt 1 ] && echo --no-cpu-baseline ) > gpurun_out/dist_c3_$r.json 2>/dev/null
  python - $r <<'PY'
import json, sys
r = sys.argv[1]
d = json.loads(open(f"gpurun_out/dist_c3_{r}.json").read().strip().splitlines()[-1])
print(r, round(d["value"], 2), "link", round(d["roofline_link"]["frac"], 3), "roof", round(d["roofline"]["frac"], 3),
      "event_check", d["roofline"].get("event_check", {}).get("achieved"), "bidir", round(d["hostlink_peak"]["bidir_gbs"], 1),
      "memcpy/step", d["memcpy_calls_per_step"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
