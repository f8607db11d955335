#!/bin/bash
# Round profile pass (one GPU): ncu launch lists (per-launch device time; DRAM
# bytes in a second pass) of the C2 / C3 decode steps and --set full captures.
# Outputs under gpurun_out/; scripts/summarize_profiles.py turns them into profiles/.
export BENCH_NO_CPU=1
# ncu serialises kernels anyway; plain stream order avoids a replay failure of a
# programmatic-dependent graph node under the profiler
export VTC_NO_PDL=1
for cfg in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$cfg.csv \
     python bench.py --config $cfg --steps 2 --warmup 1 > gpurun_out/ncu_launch_$cfg.log 2>&1; echo launch_$cfg=$?
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/dram_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 > gpurun_out/ncu_dram_$cfg.log 2>&1; echo dram_$cfg=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_stream -s 4 -c 4 \
   -o gpurun_out/full_gemv_stream python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 1 -c 1 \
   -o gpurun_out/full_attn_c3 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/ncu_full_attn.log 2>&1; echo full_attn=$?
