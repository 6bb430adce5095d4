#!/bin/bash
# One GPU-box session: build check, smoke, GPU parity tests, bench (C2 default + other configs), ncu launch list +
# full capture of the transfer kernels.  Env: SKIP_TESTS, NCU=1, WORKLOADS="c3 c4 c5".
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
python tools/show_bench.py gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
head -c 600 gpurun_out/bench_ref.json; echo
for w in ${WORKLOADS:-c3 c4 c5}; do
  timeout 900 python bench.py --workload $w --steps 30 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"
  python tools/show_bench.py gpurun_out/bench_$w.json | head -3; tail -2 gpurun_out/bench_$w.err
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 8 -c 4 -o gpurun_out/prof_staged -f \
     python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_full_staged.log 2>&1; echo "ncu full staged rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 4 -c 2 -o gpurun_out/prof_direct -f \
     python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline --mode direct > gpurun_out/ncu_full_direct.log 2>&1; echo "ncu full direct rc=$?"
fi
