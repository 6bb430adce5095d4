#!/bin/bash
# Round-2 check: build, smoke, the new ordering tests, the GPU parity suite, bench C3 (default) + C2.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 300 python -m pytest tests/test_gpu_ordering.py -x -q > gpurun_out/pytest_ordering.log 2>&1; echo "ordering rc=$?"; tail -3 gpurun_out/pytest_ordering.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for w in c3 c2 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"
  python tools/show_bench.py gpurun_out/bench_$w.json | head -3; tail -2 gpurun_out/bench_$w.err
done
