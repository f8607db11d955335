#!/bin/bash
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_GEMV_L2PF=3" "VTC_GEMV_L2PF=5" "VTC_GEMV_L2PF=8" "VTC_GEMV_L2PF=12" "VTC_X=0"; do
  env $v timeout 300 python bench.py --config c2 --steps 30 > gpurun_out/sw_c2.json 2> gpurun_out/sw_c2.err;
  python -c "import json; d=json.load(open('gpurun_out/sw_c2.json')); print('$v', round(d['value'],2), round(d['e2e']['value'],2), [round(l['us'],1) for l in d['launch_timeline']])"
done
