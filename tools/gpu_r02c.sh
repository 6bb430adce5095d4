#!/bin/bash
# Round-2: full GPU suite after the DIRECT launch defaults; C3 default + direct / mixed bench lines; ncu of the direct
# kernels alone (PCIe counters).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc=$?"; tail -2 gpurun_out/bench_default.err
for m in direct mixed; do
timeout 900 python3 bench.py --steps 20 --warmup 5 --mode $m --no-cpu-baseline > gpurun_out/bench_c3_$m.json 2> gpurun_out/bench_c3_$m.err; echo "bench $m rc=$?"; tail -2 gpurun_out/bench_c3_$m.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xfer_bulk -c 2 -o gpurun_out/prof_direct -f \
   python tools/direct_probe.py --geom c2 --focus --reps 1 > gpurun_out/ncu_direct.log 2>&1; echo "ncu direct rc=$?"
