#!/bin/bash
# Round-2 ncu evidence: the launch list of the exact default bench command, a --set full capture of the dominant
# kernel (the staged gather k_xfer_bulk<true>) inside the C3 timed loop, and the C3-sized DRAM-traffic capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_default_cmd.csv \
   python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ncu_launch_default.log 2>&1; echo "ncu launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer_bulk -s 40 -c 2 -o gpurun_out/prof_c3_loop -f \
   python3 bench.py --steps 6 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_full_loop.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_xfer_bulk -o gpurun_out/prof_traffic_c3 -f \
   python tools/traffic_probe.py c3 480 > gpurun_out/ncu_traffic_c3.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_traffic.py gpurun_out/prof_traffic_c3.ncu-rep gpurun_out/traffic_probe_c3.json gpurun_out/r02_traffic_c3.json > /dev/null 2>&1; echo "traffic json rc=$?"
