# chain boundary L2 prefetch sweep (C2)
for pf in 0 4 8 16 32; do
  VTC_CHAIN_L2PF=$pf BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/ch_$pf.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ch_$pf.json')); print('chain_pf=$pf', round(d['value'],2), round(d['e2e']['value'],1), d['kernel_times_us'])"
done
VTC_NO_CHAIN=1 BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/ch_off.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ch_off.json')); print('nochain', round(d['value'],2), round(d['e2e']['value'],1), d['kernel_times_us'])"
