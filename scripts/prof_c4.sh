#!/bin/bash
# ncu --set full of the C4 (Swin) virtual-plan kernels: fc1 GEMM, qkv gather GEMM, LayerNorm rows
export BENCH_NO_CPU=1
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
     -o gpurun_out/prof_c4_$1 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/ncu_c4_$1.log 2>&1; echo ncu_$1=$?
}
run fc1 gemm_tc_kernel 6
run qkv gemm_tc_kernel 4
run ln row_warp 2
