#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_decode_steps.py tests/test_tp.py -q -x -m gpu > gpurun_out/c2_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/c2_tests.log
export BENCH_NO_CPU=1
for i in 1 2 3; do
  timeout 300 python bench.py --config c2 --steps 30 > gpurun_out/sw_c2.json 2> gpurun_out/sw_c2.err;
  python -c "import json; d=json.load(open('gpurun_out/sw_c2.json')); print(round(d['value'],2), round(d['e2e']['value'],2), [round(l['us'],1) for l in d['launch_timeline']], round(d['roofline']['frac'],3))"
done
