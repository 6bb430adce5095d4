#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { # name env...
  n=$1; shift
  env TC_BENCH_SPANS=0 "$@" timeout 600 python bench.py --no-cpu-baseline --quick --steps 100 > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'ms', round(d['ms_per_step'],3))" 2>&1 | tail -1
}
run nohead TC_HEAD_KIB=0
run nohead_offfirst TC_HEAD_KIB=0 TC_OFFLOAD_FIRST=1
run edge1_v2_4m TC_EDGE_DIRECT=1 TC_VARIANT_D2H=2 TC_HEAD_KIB=4096
run edge1_v2_2m TC_EDGE_DIRECT=1 TC_VARIANT_D2H=2 TC_HEAD_KIB=2048
run edge1_v2_4m_offfirst TC_EDGE_DIRECT=1 TC_VARIANT_D2H=2 TC_HEAD_KIB=4096 TC_OFFLOAD_FIRST=1
run edge1_v0_4m TC_EDGE_DIRECT=1 TC_HEAD_KIB=4096
run edge3_v2_4m TC_EDGE_DIRECT=3 TC_VARIANT_D2H=2 TC_VARIANT_H2D=2 TC_HEAD_KIB=4096
run nohead_again TC_HEAD_KIB=0
TC_EDGE_DIRECT=1 TC_VARIANT_D2H=2 TC_HEAD_KIB=4096 TC_DUMP_TIMELINE=gpurun_out/tl_e1.json timeout 600 python bench.py --no-cpu-baseline --quick --steps 20 > /dev/null 2>&1
python - <<'PY'
import json
tl=json.load(open("gpurun_out/tl_e1.json"))
by={}
for s,k,a,b,n in tl: by.setdefault(s,[]).append((a,b,k,n))
for s in sorted(by)[3:7]:
    print("step",s)
    for a,b,k,n in sorted(by[s]): print("   %-20s %8.3f %8.3f  %6.1f MB" % (k,a,b,n/1e6))
PY
