#!/bin/bash
# Round-end style check: GPU tests, smoke, the default bench and the reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/rc_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/rc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/rc_bench.json').read().strip().splitlines()[-1])
print('C2', d['value'], d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'), d.get('clocks'))
for k,v in (d.get('configs') or d.get('nested') or {}).items():
    try: print(k, v.get('value'), v.get('e2e',{}).get('value') if isinstance(v.get('e2e'),dict) else None)
    except Exception as e: print(k, e)
PY
