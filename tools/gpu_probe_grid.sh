#!/bin/bash
# Device-tier probe of the TMA kernel over ring sizes (TC_TMA_RING_KIB) and grids, C2 and C5 geometry.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ring in 64 96; do
  echo "== C2 ring $ring"
  PSIZES=32,104,270,512 PVARS=3 PGRIDS='{"3":[444,888,1332,2220]}' TC_TMA_RING_KIB=$ring timeout 600 python tools/tier_probe.py 2>&1 | grep '^{'
  echo "== C5 ring $ring"
  PL=80 PH=1 PN=65536 PSIZES=32,104,270,512 PVARS=3 PGRIDS='{"3":[444,888,1332,2220]}' TC_TMA_RING_KIB=$ring timeout 600 python tools/tier_probe.py 2>&1 | grep '^{'
done
