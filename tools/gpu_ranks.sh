#!/bin/bash
# Rehearsal of the N-rank bench flow on a 1-GPU box: 2 ranks (gloo) sharing cuda:0, C2 per rank.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TC_BENCH_BACKEND=gloo TC_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 --quick > gpurun_out/bench_2ranks.json 2> gpurun_out/bench_2ranks.err
echo "2-rank rc=$?"; tail -3 gpurun_out/bench_2ranks.err; head -c 700 gpurun_out/bench_2ranks.json; echo
TC_BENCH_BACKEND=gloo TC_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 1 --impl reference > gpurun_out/bench_2ranks_ref.json 2> gpurun_out/bench_2ranks_ref.err
echo "2-rank ref rc=$?"; head -c 300 gpurun_out/bench_2ranks_ref.json; echo
