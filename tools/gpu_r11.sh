#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --peer --steps 50 --no-cpu-baseline > gpurun_out/bench_c2_peer.json 2> gpurun_out/bench_c2_peer.err; echo "bench peer rc=$?"; tail -2 gpurun_out/bench_c2_peer.err
python tools/show_bench.py gpurun_out/bench_c2_peer.json | head -4
