#!/bin/bash
# ncu --set full of C4 kernels via scripts/run_plan.py (no bench overhead)
mkdir -p gpurun_out
export VTC_NO_PDL=1
timeout 300 python scripts/run_plan.py c4 3 > gpurun_out/run_c4.log 2>&1; echo run=$?; tail -2 gpurun_out/run_c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 4 \
   -o gpurun_out/prof_c4_skinny -f python scripts/run_plan.py c4 2 > gpurun_out/ncu_c4_skinny.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 1 -c 1 \
   -o gpurun_out/prof_c4_attn -f python scripts/run_plan.py c4 2 > gpurun_out/ncu_c4_attn.log 2>&1; echo ncu2=$?
timeout 300 python bench.py --config c4 --steps 10 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo c4=$?
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(round(d['value'],1), d['kernel_times_us']); [print('   ', l) for l in d['launch_timeline']]"
