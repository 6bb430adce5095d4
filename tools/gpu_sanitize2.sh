#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SAN_VARIANT=2 timeout 1200 compute-sanitizer --tool initcheck --target-processes all --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_initcheck_simt.log 2>&1; echo "initcheck simt rc=$?"; tail -3 gpurun_out/sanitize_initcheck_simt.log
