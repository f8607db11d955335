#!/bin/bash
# ncu --set full of the C3 decode GEMMs via scripts/run_plan.py
mkdir -p gpurun_out
export VTC_NO_PDL=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 4 -c 4 \
   -o gpurun_out/prof_c3_gemm -f python scripts/run_plan.py c3 2 > gpurun_out/ncu_c3_gemm.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_c3_gemm.log
