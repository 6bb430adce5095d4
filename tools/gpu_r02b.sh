#!/bin/bash
# Round-2 evidence run: exhaustive full-size parity, the ordering tests, the driver's default bench command (C3),
# the C5 sweep line, the reference arm, a 2-rank self-launched rehearsal on one GPU (gloo), ncu launch list + full
# capture of the default command's transfer kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_ordering.py -x -q -s ${PYTEST_ARGS} > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "blocks uploaded|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -20
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc=$?"; tail -3 gpurun_out/bench_default.err
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; head -c 400 gpurun_out/bench_ref.json; echo
timeout 900 python3 bench.py --workload c5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"; tail -3 gpurun_out/bench_c5.err
TC_BENCH_BACKEND=gloo TC_BENCH_DEVICE=0 timeout 1200 python3 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_2ranks.json 2> gpurun_out/bench_2ranks.err; echo "bench 2 ranks rc=$?"; tail -3 gpurun_out/bench_2ranks.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_default.csv \
   python3 bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer -s 6 -c 2 -o gpurun_out/prof_c3 -f \
   python3 bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out
