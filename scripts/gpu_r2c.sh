#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -12 gpurun_out/pytest_gpu.log
for c in c5 c3 c4; do BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print(round(d['value'],1), d['kernel_times_us'], round(d['roofline']['frac'],3))" 2>&1 | tail -1; done
