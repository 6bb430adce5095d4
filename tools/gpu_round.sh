#!/bin/bash
# One GPU-box session: build check, smoke, GPU parity tests, bench (modes), ncu launch list + full capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
fi
for m in ${MODES:-auto direct}; do
  timeout 600 python bench.py --mode $m ${BENCH_ARGS} > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; echo "bench $m rc=$?"
  head -c 2500 gpurun_out/bench_$m.json; echo; tail -3 gpurun_out/bench_$m.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 12 -c 4 -o gpurun_out/prof_staged -f \
     python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_full_staged.log 2>&1; echo "ncu full staged rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 6 -c 2 -o gpurun_out/prof_direct -f \
     python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline --mode direct > gpurun_out/ncu_full_direct.log 2>&1; echo "ncu full direct rc=$?"
  tail -3 gpurun_out/ncu_full_direct.log
fi
