#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tma or device_tier or batches or fuzz or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
echo "== C2 default grid"; PSIZES=4,32,104,270,512 PVARS=3 PGRIDS='{"3":[0]}' timeout 600 python tools/tier_probe.py 2>&1 | grep '^{'
echo "== C5 default grid"; PL=80 PH=1 PN=65536 PSIZES=4,32,104,270,512 PVARS=3 PGRIDS='{"3":[0]}' timeout 600 python tools/tier_probe.py 2>&1 | grep '^{'
for w in c2 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 30 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1])
print('$w', round(d['value'],2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'link', round(d['roofline_link']['frac'],3), 'dev', round(d['roofline_device']['gather']['frac'],3), round(d['roofline_device']['scatter']['frac'],3), 'up', round(d['kernels']['upload_kernel']['frac'],3))
"
done
