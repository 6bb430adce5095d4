#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_auto.json 2> gpurun_out/bench_auto.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_auto.err
python tools/show_bench.py gpurun_out/bench_auto.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python tools/xfer_probe.py > gpurun_out/xfer_probe.log 2>&1; echo "probe rc=$?"; grep staged gpurun_out/xfer_probe.log
