#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5; do
  timeout 600 ncu --set full --clock-control none -k regex:k_xfer_bulk -c 4 -o gpurun_out/prof_traffic_$c -f python tools/traffic_probe.py $c > gpurun_out/ncu_traffic_$c.log 2>&1; echo "ncu traffic $c rc=$?"
done
run() { # name env...
  n=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu-baseline --quick --steps 100 > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'ms', round(d['ms_per_step'],3), 'link', round(d['roofline_link']['frac'],3))" 2>&1 | tail -1
}
run base X=1
run head16m TC_HEAD_KIB=16384
run head32m TC_HEAD_KIB=32768
run head8m TC_HEAD_KIB=8192
run base2 X=1
run head16m_2 TC_HEAD_KIB=16384
