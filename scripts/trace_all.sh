#!/bin/bash
# Device timelines (VTC_TRACE=1) + bench lines for every config. Outputs under gpurun_out/.
mkdir -p gpurun_out
export BENCH_NO_CPU=1
for cfg in ${CFGS:-c2 c3 c4 c5}; do
  VTC_TRACE=1 timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 > gpurun_out/tr_$cfg.json 2> gpurun_out/tr_$cfg.err; echo $cfg=$?
  grep -A40 "trace virtual" gpurun_out/tr_$cfg.err | head -40
  python -c "import json; d=json.load(open('gpurun_out/tr_$cfg.json')); print('$cfg', round(d['value'],1), 'mat', round(d['materialized_us'],1), d['kernel_times_us'], 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))"
done
