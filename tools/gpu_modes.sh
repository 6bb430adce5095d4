#!/bin/bash
# Bench matrix smoke: every mode / option combination completes and prints one JSON line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for args in "--workload c1" "--mode direct" "--mode staged" "--mode copy" "--mode mixed" "--peer" "--workload c5 --mode direct --steps 5"; do
  timeout 600 python bench.py $args --steps 10 --warmup 3 --no-cpu-baseline --quick > gpurun_out/m.json 2> gpurun_out/m.err
  rc=$?
  python -c "
import json
d=json.loads(open('gpurun_out/m.json').read().strip().splitlines()[-1])
print('$args', 'rc=$rc', round(d['value'],2), d['config']['xfer'], d['roofline']['kernel'] if d['roofline'] else None, round(d['roofline']['frac'],3) if d['roofline'] and d['roofline']['frac'] else None, d['steady_state']['sync_every'])
" 2>&1 | tail -1
  if [ $rc -ne 0 ]; then tail -3 gpurun_out/m.err; fi
done
