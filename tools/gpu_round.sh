#!/bin/bash
# One GPU-box session: build check, smoke, GPU parity tests, bench (modes), ncu launch list.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for m in ${MODES:-direct staged}; do
  timeout 600 python bench.py --mode $m --steps ${STEPS:-30} --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; echo "bench $m rc=$?"
  tail -c 3000 gpurun_out/bench_$m.json; tail -5 gpurun_out/bench_$m.err
done
