#!/bin/bash
# Upload-stream priority A/B on one box: the DMA pattern probe with default / high-priority upload streams, then the
# default C3 bench with the library's high-priority upload streams (default) and with TC_UP_PRIORITY=0, twice.
mkdir -p gpurun_out
for P in 0 1; do PROBE_UP_PRIORITY=$P python tools/dma_pattern_probe.py 2>&1 | head -2 | sed "s/^/prio=$P /"; done
for i in 1 2; do for P in 1 0; do
TC_UP_PRIORITY=$P timeout 600 python3 bench.py --steps 20 --warmup 5 --no-cpu-baseline --quick > gpurun_out/prio.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/prio.json').read().strip().splitlines()[-1]); print('c3 up_priority=$P', round(d['value'],2))"
done; done
