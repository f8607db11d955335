#!/bin/bash
# Quick GPU pass: parity tests + C2 bench (PDL on/off) + optional extra command.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
BENCH_NO_CPU=1 timeout 300 python bench.py > gpurun_out/q_c2.json 2> gpurun_out/q_c2.err; echo c2=$?
BENCH_NO_CPU=1 VTC_NO_PDL=1 timeout 300 python bench.py > gpurun_out/q_c2_nopdl.json 2>> gpurun_out/q_c2.err; echo c2nopdl=$?
python - <<'PY'
import json
for f in ['q_c2','q_c2_nopdl']:
    try:
        d=json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(d['value'],1), 'mat', round(d['materialized_us'],1), d['kernel_times_us'], 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))
    except Exception as e: print(f, 'ERR', e)
PY
tail -5 gpurun_out/q_c2.err
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
