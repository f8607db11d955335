#!/bin/bash
# Planner GPU pass: acceptance-1 / greedy / device oracle / boundary tests, then the cost-model calibration.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_planner.py -m gpu -q -x --durations=10 > gpurun_out/pytest_planner.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_planner.log
timeout 900 python scripts/calibrate.py > gpurun_out/calibrate.log 2>&1; echo calib=$?
tail -30 gpurun_out/calibrate.log
