# C2 knob sweep: attention CTA target (split-KV depth)
run() { env $1 BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/sw.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$1', round(d['value'],2), d['kernel_times_us'])"; }
run X=0
run VTC_ATTN_CTAS=32
run VTC_ATTN_CTAS=64
run VTC_ATTN_CTAS=96
run X=0
