# chained GEMV launch (VTC_CHAIN=1) x chain-boundary L2 prefetch sweep (C2), against separate launches
for pf in 0 4 8 16 32; do
  VTC_CHAIN=1 VTC_CHAIN_L2PF=$pf BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/ch_$pf.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ch_$pf.json')); print('chain_pf=$pf', round(d['value'],2), round(d['e2e']['value'],1), d['kernel_times_us'])"
done
BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/ch_off.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ch_off.json')); print('separate', round(d['value'],2), round(d['e2e']['value'],1), d['kernel_times_us'])"
