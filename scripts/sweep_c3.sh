run() { env $1 BENCH_NO_CPU=1 VTC_TRACE=1 timeout 600 python bench.py --config c3 2>gpurun_out/sw3.err > gpurun_out/sw3.json; python -c "import json; d=json.load(open('gpurun_out/sw3.json')); print('$1', round(d['value'],1), d['kernel_times_us'])"; grep -A11 "trace virtual" gpurun_out/sw3.err | grep "gemm_tc"; }
run X=0
run "VTC_TC_BN=256 VTC_TC_SPLITS=1"
run "VTC_TC_BN=128 VTC_TC_SPLITS=1"
