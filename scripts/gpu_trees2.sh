#!/bin/bash
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for v in "VTC_TC_TREES=1" "VTC_X=0" "VTC_TC_TREES=1" "VTC_X=0"; do
  env $v timeout 600 python bench.py --config c5 --steps 10 > gpurun_out/b_c5_$v.json 2> gpurun_out/b_c5.err; echo c5 $v=$?
  python -c "import json; d=json.load(open('gpurun_out/b_c5_$v.json')); print(round(d['value'],1), round(d['timeline_step_us'],1), d['clocks'])"
done
