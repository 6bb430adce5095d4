#!/bin/bash
# Round-2 refresh of the NEXT-1 / NEXT-3 evidence and the targeted ncu capture of the timed loop:
# Fig. 11 analogue, paced Time-Scheduler loop (100 ms and 1 s calls), C5 size sweep per mode, and a --set full capture
# of the staged gather/scatter inside the C3 timed loop (--mode staged: no calibration launches to skip over).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/fig11.py > gpurun_out/fig11.log 2>&1; echo "fig11 rc=$?"; tail -3 gpurun_out/fig11.log
timeout 600 python tools/paced.py --seconds 15 --fc-mean-ms 100 > gpurun_out/paced100.log 2>&1; echo "paced100 rc=$?"; tail -1 gpurun_out/paced100.log | head -c 600; echo
timeout 600 python tools/paced.py --seconds 15 --fc-mean-ms 1000 > gpurun_out/paced1000.log 2>&1; echo "paced1000 rc=$?"; tail -1 gpurun_out/paced1000.log | head -c 600; echo
timeout 900 python tools/sweep.py c5 --modes staged,direct > gpurun_out/sweep_c5.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/sweep_c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer_bulk -s 60 -c 2 -o gpurun_out/prof_c3_staged_loop -f \
   python3 bench.py --steps 6 --warmup 3 --quick --no-cpu-baseline --mode staged > gpurun_out/ncu_full_staged_loop.log 2>&1; echo "ncu full rc=$?"
