#!/bin/bash
# A/B: per-piece dependencies and per-handle completion events (default) vs batch-granular (TC_FINE_DEPS=0),
# interleaved, C4 / C5 / C3.  V=<tag> names the outputs.
V=${V:-v1}
mkdir -p gpurun_out
for i in 1 2; do for F in 1 0; do for w in c4 c5 c3; do
TC_FINE_DEPS=$F timeout 700 python3 bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/fd_${w}_${F}_${i}_$V.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/fd_${w}_${F}_${i}_$V.json').read().strip().splitlines()[-1]); print('$w fine=$F $i', round(d['value'],2), 'link', round(d['roofline_link']['frac'],3), 'bidir', round(d['hostlink_peak']['bidir_gbs'],1), 'after', round(d['hostlink_peak_after']['bidir_gbs'],1), d['config']['step'][160:215])"
done; done; done
