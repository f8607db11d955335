#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_gpu_fmha.py -q -x -k "skinny or swin or c3k2 or c4 or window" > gpurun_out/c4_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/c4_tests.log
export BENCH_NO_CPU=1
timeout 300 python bench.py --config c4 --steps 10 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo c4=$?
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/full_tests.log 2>&1; echo full=$?; tail -3 gpurun_out/full_tests.log
