#!/bin/bash
# same-box A/B of two builds of libvtc.so: libvtc_head.so vs libvtc_new.so
export BENCH_NO_CPU=1
L=paper_2604_09558_b200
for v in head new head new; do
  cp $L/libvtc_$v.so $L/libvtc.so
  timeout 300 python bench.py --config ${CFG:-c2} --steps ${STEPS:-30} > gpurun_out/ab.json 2> gpurun_out/ab.err;
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['value'],2), [round(l['us'],1) for l in d['launch_timeline']])"
done
