#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or llama" 2>&1 | tail -1
for c in 64 128 296 600; do
  VTC_ATTN_CTAS=$c BENCH_NO_CPU=1 VTC_TRACE=1 timeout 300 python bench.py --steps 10 2>gpurun_out/sa.err > gpurun_out/sa.json
  echo "ctas=$c bench=$(python -c "import json; print(round(json.load(open('gpurun_out/sa.json'))['value'],1))")"
  grep -A4 "trace virtual" gpurun_out/sa.err | grep -E "attn|eltwise" | cut -c1-130
done
