#!/bin/bash
# Retire-ladder study: refused cycles retried after tc_retire (then tc_sync).  C3 lag 1 vs 2; C4 / C5 drained vs
# retire-each lag 1 (and 2); interleaved, two rounds.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
show() { python - "$1" <<'PY'
import json, re, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
m = re.search(r"\((\d+) of (\d+) steps needed the retire, (\d+) the sync\)", d["config"]["step"])
print(sys.argv[1].split("/")[-1], round(d["value"], 2), "link", round(d["roofline_link"]["frac"], 3),
      "ladder/sync", m.groups()[:1] + m.groups()[2:] if m else "drained", "bidir", round(d["hostlink_peak"]["bidir_gbs"], 1))
PY
}
for r in 1 2; do
  for a in "c3 each 1" "c3 each 2" "c4 sync 1" "c4 each 1" "c4 each 2" "c5 sync 1" "c5 each 1"; do
    set -- $a
    f=gpurun_out/ladder_$1_$2_$3_r$r.json
    timeout 900 python3 bench.py --workload $1 --steps 20 --warmup 5 --retire $2 --retire-lag $3 --no-cpu-baseline --no-sweep > $f 2>/dev/null
    show $f
  done
done
