#!/bin/bash
# Full-size parity in the bench's configuration + bench lines in both retirement modes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or retire" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for w in c2 c3 c4 c5; do
 for r in each sync; do
  timeout 900 python bench.py --workload $w --retire $r --steps 40 --no-cpu-baseline > gpurun_out/b_${w}_$r.json 2> gpurun_out/b_${w}_$r.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_${w}_$r.json').read().strip().splitlines()[-1])
print('$w $r', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'link', round(d['roofline_link']['frac'],3), 'dom', round(d['roofline']['frac'],3), 'drain', d['per_cycle_drain'] and round(d['per_cycle_drain']['value'],2), 'bidir', round(d['hostlink_peak']['bidir_gbs'],1))
" 2>&1 | tail -1
 done
done
