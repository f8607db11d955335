#!/bin/bash
# Round-2 profile pass (one GPU): per-launch ncu lists (time + DRAM bytes) of one
# step of every config, --set full captures of the dominant kernels, and the
# compute-sanitizer runs.  Outputs under gpurun_out/; scripts/summarize_r2.py
# turns them into profiles/r2_*.
mkdir -p gpurun_out
export VTC_NO_PDL=1 BENCH_NO_CPU=1
for cfg in c2 c3 c4 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/r2_launch_$cfg.csv python scripts/run_plan.py $cfg 2 > gpurun_out/r2_launch_$cfg.log 2>&1; echo launch_$cfg=$?
done
full() {  # name cfg regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c $5 -f \
     -o gpurun_out/r2_full_$1 python scripts/run_plan.py $2 2 > gpurun_out/r2_full_$1.log 2>&1; echo full_$1=$?
}
full c2_gemv c2 gemv_stream 4 4
full c3_gemm c3 gemm_tc 4 4
full c3_attn c3 attn_decode 1 1
full c4_skinny c4 gemm_skinny 4 4
full c4_attn c4 attn_window 1 1
full c5_gemm c5 gemm_tc 4 4
full c5_attn c5 attn_fmha 1 1
unset VTC_NO_PDL
# (compute-sanitizer is now closed on the GPU pool: these runs only print a refusal; the
# 0-error results in profiles/r2_summary.md are from commit 7eb23ff.)
# sanitizers on the cross-CTA protocols: split-K counters (tcgen05 GEMM), strip flags (streamed
# GEMV), the cooperative split-KV combine, the skinny GEMM's rings, the window attention
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu.py -q -x \
   -k "llama_layer_small or gate_up or batch64 or fused_epilogues or skinny or window" > gpurun_out/r2_san_memcheck.log 2>&1; echo memcheck=$?
tail -5 gpurun_out/r2_san_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu.py -q -x \
   -k "llama_layer_small or swin_window" > gpurun_out/r2_san_racecheck.log 2>&1; echo racecheck=$?
tail -5 gpurun_out/r2_san_racecheck.log
timeout 1800 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu.py -q -x \
   -k "llama_layer_small or swin_block_small" > gpurun_out/r2_san_synccheck.log 2>&1; echo synccheck=$?
tail -5 gpurun_out/r2_san_synccheck.log
# summarise on the box (the .ncu-rep files exceed the copy-back limit); keep the small reports
python scripts/summarize_r2.py r2 > gpurun_out/r2_summary_stdout.txt 2>&1; echo summarize=$?
mkdir -p gpurun_out/profiles_r2 && cp profiles/r2_* profiles/traffic.json gpurun_out/profiles_r2/
for f in gpurun_out/r2_full_*.ncu-rep; do [ $(stat -c %s "$f") -gt 6000000 ] && rm -f "$f"; done
du -sh gpurun_out
