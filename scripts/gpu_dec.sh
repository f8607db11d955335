#!/bin/bash
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for v in "VTC_ATTN_L2PF=0" "VTC_ATTN_L2PF=1"; do
  env $v timeout 300 python bench.py --config c2 --steps 20 > gpurun_out/b_c2_$v.json 2> gpurun_out/b_c2.err; echo c2 $v=$?
  python -c "import json; d=json.load(open('gpurun_out/b_c2_$v.json')); print(round(d['value'],2), d['kernel_times_us'], d['e2e']['value']); [print('   ', l) for l in d['launch_timeline']]"
done
for v in "VTC_DECODE_BN=128" "VTC_DECODE_BN=256"; do
  env $v timeout 300 python bench.py --config c3 --steps 10 > gpurun_out/b_c3_$v.json 2> gpurun_out/b_c3.err; echo c3 $v=$?
  python -c "import json; d=json.load(open('gpurun_out/b_c3_$v.json')); print(round(d['value'],2), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
done
