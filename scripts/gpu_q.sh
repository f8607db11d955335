#!/bin/bash
# quick: selected GPU tests ($TESTS) + one bench config ($CFG)
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -q -x > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q_tests.log; fi
for c in $CFG; do BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print(round(d['value'],1), d['kernel_times_us'], round(d['roofline']['frac'],3))" 2>&1 | tail -1; done
