#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_decode_steps.py -q -x > gpurun_out/coop_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/coop_tests.log
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_NO_COOP_REDUCE=1" "VTC_X=0" "VTC_NO_COOP_REDUCE=1"; do
  env $v timeout 300 python bench.py --config c3 --steps 10 > gpurun_out/sw_c3.json 2> gpurun_out/sw_c3.err;
  python -c "import json; d=json.load(open('gpurun_out/sw_c3.json')); print('$v', round(d['value'],2), [round(l['us'],1) for l in d['launch_timeline']])"
done
