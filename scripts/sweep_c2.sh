# C2 knob sweep: GEMV ring depth
run() { env $1 BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/sw.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$1', round(d['value'],2), d['kernel_times_us'])"; }
run X=0
run VTC_GEMV_STAGES=4
run VTC_GEMV_STAGES=5
run "VTC_GEMV_STAGES=4 VTC_GEMV_PRE=2"
run X=0
