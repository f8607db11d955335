for pf in 0 4 8 16 32 64; do
  BENCH_NO_CPU=1 VTC_GEMV_L2PF=$pf timeout 300 python bench.py > gpurun_out/pf_$pf.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pf_$pf.json')); print('pf=$pf', round(d['value'],2), d['kernel_times_us'], round(d['roofline']['frac'],3))"
done
BENCH_NO_CPU=1 VTC_TRACE=1 VTC_GEMV_L2PF=16 timeout 300 python bench.py 2>&1 >/dev/null | grep -A7 "trace virtual"
