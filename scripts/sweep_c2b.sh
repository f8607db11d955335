#!/bin/bash
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_ATTN_CTAS=148" "VTC_ATTN_CTAS=444" "VTC_GEMV_STAGES=4" "VTC_GEMV_PRE=2" "VTC_ATTN_L2PF=0" "VTC_X=0"; do
  env $v timeout 300 python bench.py --config c2 --steps 30 > gpurun_out/sw_c2.json 2> gpurun_out/sw_c2.err; 
  python -c "import json; d=json.load(open('gpurun_out/sw_c2.json')); print('$v', round(d['value'],2), round(d['e2e']['value'],2), [round(l['us'],1) for l in d['launch_timeline']])"
done
