#!/bin/bash
# Slow-box hunt: a quick C3 line; if it is below 97 GB/s, A/B the upload-stream priority and the staging halves on
# this box (the loop's H2D shortfall seen on some boxes).
mkdir -p gpurun_out
timeout 600 python3 bench.py --steps 12 --warmup 3 --no-cpu-baseline --quick > gpurun_out/sb0.json 2>/dev/null
v=$(python -c "import json; print(round(json.loads(open('gpurun_out/sb0.json').read().strip().splitlines()[-1])['value'],2))")
echo "c3 quick: $v"
if python -c "import sys; sys.exit(0 if $v < 97 else 1)"; then
  for i in 1 2; do
    for cfg in "TC_UP_PRIORITY=1" "TC_UP_PRIORITY=0" "TC_STAGING_HALVES=0" "TC_FINE_DEPS=0" "TC_STAGING_MIB=4096"; do
      env $cfg timeout 600 python3 bench.py --steps 12 --warmup 3 --no-cpu-baseline --quick > gpurun_out/sb.json 2>/dev/null
      python -c "import json; print('$cfg', round(json.loads(open('gpurun_out/sb.json').read().strip().splitlines()[-1])['value'],2))"
    done
  done
  python tools/dma_pattern_probe.py 2>&1 | head -2
fi
