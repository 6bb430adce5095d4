#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tma or device_tier" > gpurun_out/pytest_tma.log 2>&1; echo "pytest tma rc=$?"; tail -5 gpurun_out/pytest_tma.log
timeout 900 python tools/xfer_probe.py > gpurun_out/xfer_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/xfer_probe.log | tail -40
