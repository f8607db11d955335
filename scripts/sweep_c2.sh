# C2: shared-memory carveout A/B (max carveout for every kernel vs the driver default)
run() { env $1 BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/sw.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$1', round(d['value'],2), round(d['e2e']['value'],2), d['kernel_times_us'])"; }
run X=0
run VTC_DEFAULT_CARVEOUT=1
run "VTC_GEMV_STAGES=2 VTC_ATTN_CTAS=148"
run X=0
