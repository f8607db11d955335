#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "4 2" "3 1" "6 2" "2 1" "4 4" "3 3"; do
  set -- $cfg
  VTC_GEMV_STAGES=$1 VTC_GEMV_PRE=$2 BENCH_NO_CPU=1 VTC_TRACE=1 timeout 300 python bench.py --l2 none --steps 10 2>gpurun_out/sw.err > gpurun_out/sw.json
  echo "stages=$1 pre=$2 bench=$(python -c "import json; print(round(json.load(open('gpurun_out/sw.json'))['value'],1))")"
  grep -A9 "trace virtual" gpurun_out/sw.err | grep -E "total|gemv" | cut -c1-120
done
