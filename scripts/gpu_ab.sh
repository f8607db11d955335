#!/bin/bash
export BENCH_NO_CPU=1
for v in $AB; do
  env $v timeout 600 python bench.py --config ${CFG:-c5} --steps 10 > gpurun_out/ab.json 2> gpurun_out/ab.err;
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['value'],1), [round(l['us'],1) for l in d['launch_timeline']])"
done
