#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TC_DUMP_TIMELINE=gpurun_out/tl_staged.json timeout 600 python bench.py --no-cpu-baseline --quick --steps 20 > gpurun_out/bench_tl.json 2> gpurun_out/bench_tl.err; echo "bench rc=$?"
python - <<'PY'
import json
tl=json.load(open("gpurun_out/tl_staged.json"))
by={}
for s,k,a,b,n in tl: by.setdefault(s,[]).append((a,b,k,n))
for s in sorted(by)[:6]:
    print("step",s)
    for a,b,k,n in sorted(by[s]): print("   %-15s %8.3f %8.3f  %6.1f MB" % (k,a,b,n/1e6))
PY
