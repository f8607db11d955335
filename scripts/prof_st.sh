#!/bin/bash
mkdir -p gpurun_out
export VTC_NO_PDL=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_stream -s 3 -c 3 \
   -o gpurun_out/prof_c3_stream -f python scripts/run_plan.py c3 2 > gpurun_out/ncu_c3_stream.log 2>&1; echo ncu=$?
