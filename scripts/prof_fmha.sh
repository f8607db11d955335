#!/bin/bash
# fmha parity + C5-size attention-only timing + one ncu --set full capture of the kernel.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x -s > gpurun_out/fmha.log 2>&1; echo fmha=$?
grep -E "rel err|passed|failed|Error" gpurun_out/fmha.log | head -20
timeout 300 python scripts/fmha_bench.py > gpurun_out/fmha_bench.log 2>&1; echo fb=$?; cat gpurun_out/fmha_bench.log | tail -5
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fmha -c 1 -o gpurun_out/prof_fmha -f python scripts/fmha_bench.py --once > gpurun_out/ncu_fmha.log 2>&1; echo ncu=$?
fi
