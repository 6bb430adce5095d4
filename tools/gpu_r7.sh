#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "piece or unbuffered or c1 or fuzz" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_auto.json 2> gpurun_out/bench_auto.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_auto.err
python tools/show_bench.py gpurun_out/bench_auto.json
python -c "import json; d=json.loads(open('gpurun_out/bench_auto.json').read().strip().splitlines()[-1]); print(json.dumps(d['timeline']))"
timeout 900 python tools/fig11.py > gpurun_out/fig11.log 2>&1; echo "fig11 rc=$?"; cat gpurun_out/fig11.log | tail -20
