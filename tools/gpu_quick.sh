#!/bin/bash
# Quick GPU check: smoke, a parity subset, the C2 bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "${PYTEST_K:-c1 or fuzz or device_tier or peer}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_c2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1])
print('c2', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'launches', d['roofline'].get('bytes_per_launch'), 'link', round(d['roofline_link']['frac'],3), 'dev', round(d['roofline_device']['gather']['frac'],3), round(d['roofline_device']['scatter']['frac'],3), d['kernels']['offload_kernel']['launches'])
"
