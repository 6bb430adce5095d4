#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for e in 1 0; do
TC_EDGE_DIRECT=$e TC_DUMP_TIMELINE=gpurun_out/tl_edge$e.json timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_edge$e.json 2> gpurun_out/bench_edge$e.err; echo "bench edge$e rc=$?"; tail -2 gpurun_out/bench_edge$e.err
python tools/show_bench.py gpurun_out/bench_edge$e.json
done
python - <<'PY'
import json
tl=json.load(open("gpurun_out/tl_edge1.json"))
by={}
for s,k,a,b,n in tl: by.setdefault(s,[]).append((a,b,k,n))
for s in sorted(by)[3:7]:
    print("step",s)
    for a,b,k,n in sorted(by[s]): print("   %-20s %8.3f %8.3f  %6.1f MB" % (k,a,b,n/1e6))
PY
