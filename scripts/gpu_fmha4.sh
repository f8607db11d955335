#!/bin/bash
mkdir -p gpurun_out
for e in 0 -1; do echo emu=$e; VTC_FMHA_EMU=$e timeout 300 python scripts/fmha_bench.py; VTC_FMHA_EMU=$e timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x -s 2>&1 | grep -E "rel err|passed|failed"; done
