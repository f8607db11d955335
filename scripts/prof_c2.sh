#!/bin/bash
# ncu --set full captures of the C2 decode-layer kernels (one launch each, after warm-up).
export BENCH_NO_CPU=1
mkdir -p gpurun_out
TAG=${TAG:-r1}
for k in ew_kernel combine_kernel attn_kernel gemv_kernel ${EXTRA_KERNELS}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 8 -c 1 \
     -o gpurun_out/prof_${TAG}_$k python bench.py --steps 2 --warmup 1 ${BENCH_ARGS} > gpurun_out/ncu_${TAG}_$k.log 2>&1; echo ncu_$k=$?
done
