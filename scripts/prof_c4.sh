#!/bin/bash
# ncu --set full of one C4 (Swin) virtual-plan kernel: prof_c4.sh NAME KERNEL_REGEX SKIP
# (defaults: the fc1 GEMM)
export BENCH_NO_CPU=1
name=${1:-fc1}; regex=${2:-gemm_tc_kernel}; skip=${3:-6}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c 1 \
   -o gpurun_out/prof_c4_$name python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/ncu_c4_$name.log 2>&1; echo ncu_$name=$?
