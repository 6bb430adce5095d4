#!/bin/bash
# A/B: item-aligned piece cuts (default, TC_MIN_PIECE_MIB=64) vs unaligned (TC_MIN_PIECE_MIB=100000), interleaved:
# resume latency (tools/resume_latency.py) and the bench lines of C3 / C5 / C4 / C2.  V=<tag> names the outputs.
V=${V:-v1}
mkdir -p gpurun_out
for M in 64 100000; do TC_MIN_PIECE_MIB=$M python tools/resume_latency.py 12 | sed "s/^{/{\"min_piece_mib\": $M, /"; done > gpurun_out/align_resume_$V.jsonl
cat gpurun_out/align_resume_$V.jsonl
for i in 1 2; do for M in 64 100000; do for w in c3 c5 c4 c2; do
TC_MIN_PIECE_MIB=$M timeout 700 python3 bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/al_${w}_${M}_${i}_$V.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/al_${w}_${M}_${i}_$V.json').read().strip().splitlines()[-1]); print('$w min_piece=$M $i', round(d['value'],2), 'link', round(d['roofline_link']['frac'],3), 'bidir', round(d['hostlink_peak']['bidir_gbs'],1), 'memcpy/step', round(d['memcpy_calls_per_step'],1), 'launches', d['gpu_launches'])"
done; done; done
