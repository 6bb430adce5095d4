#!/bin/bash
# Kernel-variant session: GPU parity, device-tier probe, bench per mode/variant.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/tier_probe.py > gpurun_out/tier_probe.log 2>&1; echo "tier rc=$?"
for v in ${VARS:-0 2 3}; do
  TC_VARIANT_DEV=$v timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_staged_v$v.json 2> gpurun_out/bench_staged_v$v.err; echo "bench staged v$v rc=$?"
  python tools/show_bench.py gpurun_out/bench_staged_v$v.json
done
for m in ${BMODES:-mixed direct}; do
  TC_VARIANT_DEV=3 timeout 600 python bench.py --no-cpu-baseline --steps 50 --mode $m > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; echo "bench $m rc=$?"
  python tools/show_bench.py gpurun_out/bench_$m.json
done
