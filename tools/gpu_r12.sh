#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_c2.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['config']['numa'], d['roofline']['frac'], d['roofline_link']['frac'])"
for c in c3 c4; do
  timeout 600 ncu --set full --clock-control none -k regex:k_xfer_bulk -c 4 -o gpurun_out/prof_traffic_$c -f python tools/traffic_probe.py $c > gpurun_out/ncu_traffic_$c.log 2>&1; echo "ncu traffic $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 8 -c 4 -o gpurun_out/prof_staged -f \
     python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_full_staged.log 2>&1; echo "ncu full staged rc=$?"
