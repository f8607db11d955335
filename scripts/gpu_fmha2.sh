#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x > gpurun_out/fmha.log 2>&1; echo fmha=$?; tail -1 gpurun_out/fmha.log
timeout 300 python scripts/fmha_bench.py; VTC_TRACE=1 timeout 300 python scripts/fmha_bench.py
FMHA_CAUSAL=0 timeout 300 python scripts/fmha_bench.py
