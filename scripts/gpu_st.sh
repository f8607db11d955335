#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "stream_tc" > gpurun_out/st_tests.log 2>&1; echo st=$?; tail -15 gpurun_out/st_tests.log
export BENCH_NO_CPU=1
timeout 300 python bench.py --config c3 --steps 10 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo c3=$?
python -c "import json; d=json.load(open('gpurun_out/b_c3.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
tail -3 gpurun_out/b_c3.err
