#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x > gpurun_out/fmha.log 2>&1; echo fmha=$?; tail -1 gpurun_out/fmha.log
for e in 0 2 3 4; do echo emu=$e; VTC_FMHA_EMU=$e timeout 300 python scripts/fmha_bench.py; done
VTC_TRACE=1 timeout 300 python scripts/fmha_bench.py
VTC_FMHA_EMU=4 timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x 2>&1 | tail -1
