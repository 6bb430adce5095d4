#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tma or device_tier or batches or c1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for ring in 32 64 96; do
  echo "== C5 geometry ring $ring"
  PL=80 PH=1 PN=65536 PSIZES=4,32,104,512 PVARS=3 PGRIDS='{"3":[296,444,592]}' TC_TMA_RING_KIB=$ring timeout 600 python tools/tier_probe.py 2>&1 | tail -12
done
echo "== C5 geometry tile / v1"
PL=80 PH=1 PN=65536 PSIZES=4,104,512 PVARS=1,2 PGRIDS='{"1":[148],"2":[1184,2368]}' timeout 600 python tools/tier_probe.py 2>&1 | tail -9
for ring in 32 96; do
  echo "== C2 geometry ring $ring"
  PSIZES=4,32,104,512 PVARS=3 PGRIDS='{"3":[296,444,592]}' TC_TMA_RING_KIB=$ring timeout 600 python tools/tier_probe.py 2>&1 | tail -12
done
echo "== C2 geometry default ring"
PSIZES=4,32,104,512 PVARS=3 PGRIDS='{"3":[296,444]}' timeout 600 python tools/tier_probe.py 2>&1 | tail -8
