#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_fullsize.py -q -x -k "skinny or swin or c3k2 or c4" > gpurun_out/c4_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/c4_tests.log
export BENCH_NO_CPU=1
timeout 300 python bench.py --config c4 --steps 10 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo c4=$?
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
if [ -n "$NCU" ]; then
VTC_NO_PDL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 4 \
   -o gpurun_out/prof_c4_skinny -f python scripts/run_plan.py c4 2 > gpurun_out/ncu_c4_skinny.log 2>&1; echo ncu=$?
fi
