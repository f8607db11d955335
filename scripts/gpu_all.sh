#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -x -m gpu > gpurun_out/all_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/all_tests.log
export BENCH_NO_CPU=1
for c in ${CFGS:-c2 c3 c5}; do
  timeout 600 python bench.py --config $c --steps 10 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo $c=$?
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['value'],1), [round(l['us'],1) for l in d['launch_timeline']])"
done
