#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "cta_pair" > gpurun_out/cp_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/cp_tests.log
export BENCH_NO_CPU=1
for v in "VTC_X=0" "VTC_GEMM_CTA_PAIR=1"; do
  env $v timeout 240 python bench.py --config c5 --steps 5 > gpurun_out/b_c5_$v.json 2> gpurun_out/b_c5.err; echo c5 $v=$?
  python -c "import json; d=json.load(open('gpurun_out/b_c5_$v.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
done
