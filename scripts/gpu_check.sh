#!/bin/bash
# One GPU-box pass: parity tests, smoke, every bench config, the reference arm.  Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2=$?
for c in c1 c3 c4 c5; do
  BENCH_NO_CPU=${NOCPU:-} timeout 900 python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench_ref=$?
tail -3 gpurun_out/pytest_gpu.log
