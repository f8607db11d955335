#!/bin/bash
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_ATTN_CTAS=2048" "VTC_ATTN_CTAS=3584" "VTC_ATTN_CTAS=5120" "VTC_X=0"; do
  env $v timeout 300 python bench.py --config c3 --steps 10 > gpurun_out/sw_c3.json 2> gpurun_out/sw_c3.err; 
  python -c "import json; d=json.load(open('gpurun_out/sw_c3.json')); print('$v', round(d['value'],2), [round(l['us'],1) for l in d['launch_timeline']])"
done
