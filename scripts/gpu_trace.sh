#!/bin/bash
# parity tests + C2 timeline + C2 bench line
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
BENCH_NO_CPU=1 VTC_TRACE=1 timeout 300 python bench.py ${BENCH_ARGS} > gpurun_out/t_c2.json 2>gpurun_out/t_c2.err; echo trace=$?
grep -A12 "trace virtual" gpurun_out/t_c2.err
BENCH_NO_CPU=1 timeout 300 python bench.py ${BENCH_ARGS} > gpurun_out/q_c2.json 2>gpurun_out/q_c2.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/q_c2.json')); print(d['value'], 'mat', d['materialized_us'], d['kernel_times_us'], d['roofline']['frac'])"
