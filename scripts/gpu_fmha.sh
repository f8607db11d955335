#!/bin/bash
# tcgen05 flash attention: parity, then the C5 layer timing, then the planner tests.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x -s > gpurun_out/fmha.log 2>&1; echo fmha=$?
grep -E "rel err|passed|failed|Error" gpurun_out/fmha.log | head -20
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "prefill" > gpurun_out/prefill.log 2>&1; echo prefill=$?; tail -3 gpurun_out/prefill.log
BENCH_NO_CPU=1 timeout 600 python bench.py --config c5 --steps 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['value'], d['kernel_times_us'], d['roofline'])" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_planner.py -q -x > gpurun_out/pytest_planner.log 2>&1; echo planner=$?; tail -3 gpurun_out/pytest_planner.log
