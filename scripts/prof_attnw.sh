#!/bin/bash
mkdir -p gpurun_out
export VTC_NO_PDL=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_window -s 1 -c 1 \
   -o gpurun_out/prof_c4_attnw -f python scripts/run_plan.py c4 2 > gpurun_out/ncu_c4_attnw.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_c4_attnw.log
