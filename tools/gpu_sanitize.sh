#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py (every kernel path).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "many_seeds or concatenate" > gpurun_out/pytest_new.log 2>&1; echo "pytest new rc=$?"; tail -3 gpurun_out/pytest_new.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --target-processes all --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "sanitizer $t rc=$?"; tail -3 gpurun_out/sanitize_$t.log
done
SAN_VARIANT=2 timeout 1200 compute-sanitizer --tool initcheck --target-processes all --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_initcheck_simt.log 2>&1; echo "initcheck simt rc=$?"; tail -1 gpurun_out/sanitize_initcheck_simt.log
