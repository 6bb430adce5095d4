#!/bin/bash
# C3 loop study: retire lag 1 / 2 / 3 and staging 1 / 4 GiB, interleaved, two rounds.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
 for cfg in "1 1024" "2 1024" "3 1024" "1 4096" "2 4096"; do
  set -- $cfg
  TC_STAGING_MIB=$2 timeout 600 python3 bench.py --steps 30 --warmup 5 --retire each --retire-lag $1 --no-cpu-baseline > gpurun_out/c3_lag$1_stg$2_r$r.json 2>/dev/null
  python - <<PY
import json
d=json.loads(open("gpurun_out/c3_lag$1_stg$2_r$r.json").read().strip().splitlines()[-1])
print("lag $1 staging $2 run $r:", round(d["value"],2), "link", round(d["roofline_link"]["frac"],3), "drains", d["config"]["step"].split("(")[2][:20], "bidir", round(d["hostlink_peak"]["bidir_gbs"],1))
PY
 done
done
