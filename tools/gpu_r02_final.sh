#!/bin/bash
# Round-2 evidence pass on one box: build + smoke, the whole GPU suite, the driver's default bench command (C3),
# every other config's default line, the oracle arm, and the ncu launch list + --set full capture of the default
# command's dominant kernel.  V=<tag> names the outputs.
V=${V:-final}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$V.log
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$V.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default_$V.json 2> gpurun_out/bench_default_$V.err; echo "bench default rc=$?"
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err; echo "bench ref rc=$?"
for w in c2 c4 c5; do
  timeout 900 python3 bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_${w}_$V.json 2> gpurun_out/bench_${w}_$V.err; echo "bench $w rc=$?"
done
python - <<PY
import json
for n in ("default", "c2", "c4", "c5", "ref"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{n}_$V.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(n, "ERR", e); continue
    if n == "ref":
        print(n, round(d["value"], 3)); continue
    print(n, d["config"]["workload"][:3], round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "link", round(d["roofline_link"]["frac"], 3),
          "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "bidir", round(d["hostlink_peak"]["bidir_gbs"], 1),
          "cpu", d["cpu_baseline"] and round(d["cpu_baseline"]["value"], 3), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
if [ -n "$NCU" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_default_cmd_$V.csv \
   python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ncu_launch_default_$V.log 2>&1; echo "ncu launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xfer_bulk -s 60 -c 2 -o gpurun_out/prof_c3_loop_$V -f \
   python3 bench.py --steps 6 --warmup 3 --quick --no-cpu-baseline --mode staged > gpurun_out/ncu_full_loop_$V.log 2>&1; echo "ncu full rc=$?"
fi
