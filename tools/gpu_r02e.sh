#!/bin/bash
# Multi-rank rehearsal on one GPU (gloo): the self-launched 4- and 8-rank flows of bench.py on the north_star
# partition (C4 head-sharded, G = N), every rank on GPU 0.  Plumbing check, not a scaling number.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
free -g | head -2; nproc
TC_BENCH_BACKEND=gloo TC_BENCH_DEVICE=0 timeout 1200 python3 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_4ranks.json 2> gpurun_out/bench_4ranks.err; echo "4 ranks rc=$?"; tail -3 gpurun_out/bench_4ranks.err
TC_BENCH_BACKEND=gloo TC_BENCH_DEVICE=0 timeout 1500 python3 bench.py --gpus 8 --steps 10 --warmup 3 --quick > gpurun_out/bench_8ranks.json 2> gpurun_out/bench_8ranks.err; echo "8 ranks rc=$?"; tail -3 gpurun_out/bench_8ranks.err
timeout 900 python3 bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
