#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b100_$i.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b100_$i.json').read().strip().splitlines()[-1]); print('100 steps', round(d['value'],2), round(d['roofline_link']['frac'],3), round(d['ms_per_step'],3), d['hostlink_peak']['bidir_gbs'])"
done
timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/b50.json 2> /dev/null
python -c "import json; d=json.loads(open('gpurun_out/b50.json').read().strip().splitlines()[-1]); print('50 steps', round(d['value'],2), round(d['roofline_link']['frac'],3), round(d['ms_per_step'],3))"
TC_AUTO_DIRECT_KIB=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b100_nodirect.json 2> /dev/null
python -c "import json; d=json.loads(open('gpurun_out/b100_nodirect.json').read().strip().splitlines()[-1]); print('100 steps no small-direct', round(d['value'],2), round(d['roofline_link']['frac'],3), round(d['ms_per_step'],3))"
