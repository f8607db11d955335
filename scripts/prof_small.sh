export BENCH_NO_CPU=1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"ew_kernel" -s 2 -c 1 -o gpurun_out/prof_ew python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_ew.log 2>&1; echo ncu_ew=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"combine" -s 1 -c 1 -o gpurun_out/prof_comb python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_comb.log 2>&1; echo ncu_comb=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemv_tma" -s 2 -c 1 -o gpurun_out/prof_tma python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_tma.log 2>&1; echo ncu_tma=$?
grep -E "ERROR" gpurun_out/ncu_*.log | head
