#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TC_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --quick --steps 20 > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err; echo "bench trace rc=$?"
tail -8 gpurun_out/bench_trace.err
timeout 900 python tools/xfer_probe.py > gpurun_out/xfer_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/xfer_probe.log
