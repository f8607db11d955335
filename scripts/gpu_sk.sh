#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "skinny or fused_epilogues or prefill or c3k2" > gpurun_out/sk_tests.log 2>&1; echo sk=$?; tail -15 gpurun_out/sk_tests.log
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/full_tests.log 2>&1; echo full=$?; tail -5 gpurun_out/full_tests.log
export BENCH_NO_CPU=1
for c in ${CFGS:-c4 c5}; do timeout 600 python bench.py --config $c --steps 10 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo $c=$?
python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['value'],1), d['kernel_times_us'], round(d['roofline']['frac'],3)); [print('   ', l) for l in d['launch_timeline']]"; done
