#!/bin/bash
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_TC_TREES=1"; do
  env $v timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/b_c5_$v.json 2> gpurun_out/b_c5.err; echo c5 $v=$?
  python -c "import json; d=json.load(open('gpurun_out/b_c5_$v.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
done
