#!/bin/bash
# ncu --set full of selected kernels of the C2 bench: KERNELS="ew_kernel attn_decode" TAG=x
export BENCH_NO_CPU=1
for k in ${KERNELS}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 4 -c 1 \
     -o gpurun_out/prof_${TAG}_$k python bench.py --steps 2 --warmup 1 ${BENCH_ARGS} > gpurun_out/ncu_${TAG}_$k.log 2>&1; echo ncu_$k=$?
done
