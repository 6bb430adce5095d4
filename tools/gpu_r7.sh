#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "copy or c1 or batches" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
run() { # name env...
  n=$1; shift
  env TC_BENCH_SPANS=0 "$@" timeout 600 python bench.py --no-cpu-baseline --quick --steps 100 > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'ms', round(d['ms_per_step'],3), d['gpu_launches'])" 2>&1 | tail -1
}
run staged_nohead TC_HEAD_KIB=0
run copy TC_AUTO_D2H=3 TC_AUTO_H2D=3
run copy_d2h TC_AUTO_D2H=3 TC_HEAD_KIB=0
run copy_h2d TC_AUTO_H2D=3 TC_HEAD_KIB=0
run copy_nobatch TC_AUTO_D2H=3 TC_AUTO_H2D=3 TC_BATCH_MEMCPY=0
run staged_nohead2 TC_HEAD_KIB=0
for w in c3 c5; do
  TC_BENCH_SPANS=0 TC_HEAD_KIB=0 timeout 600 python bench.py --no-cpu-baseline --quick --steps 30 --workload $w > gpurun_out/b_${w}_staged.json 2>gpurun_out/b_${w}_staged.err
  TC_BENCH_SPANS=0 TC_AUTO_D2H=3 TC_AUTO_H2D=3 timeout 600 python bench.py --no-cpu-baseline --quick --steps 30 --workload $w > gpurun_out/b_${w}_copy.json 2>gpurun_out/b_${w}_copy.err
  for m in staged copy; do python -c "import json; d=json.loads(open('gpurun_out/b_${w}_$m.json').read().strip().splitlines()[-1]); print('$w $m', round(d['value'],2), 'ms', round(d['ms_per_step'],3))" 2>&1 | tail -1; done
done
TC_AUTO_D2H=3 TC_AUTO_H2D=3 TC_DUMP_TIMELINE=gpurun_out/tl_copy.json timeout 600 python bench.py --no-cpu-baseline --quick --steps 20 > /dev/null 2>&1
python - <<'PY'
import json
tl=json.load(open("gpurun_out/tl_copy.json"))
by={}
for s,k,a,b,n in tl: by.setdefault(s,[]).append((a,b,k,n))
for s in sorted(by)[3:6]:
    print("step",s)
    for a,b,k,n in sorted(by[s]): print("   %-20s %8.3f %8.3f  %6.1f MB" % (k,a,b,n/1e6))
PY
