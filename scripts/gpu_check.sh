#!/bin/bash
# One GPU-box pass: parity tests, benches, ncu launch list.  Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2=$?
timeout 600 python bench.py --config c1 --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1=$?
timeout 900 python bench.py --config c3 --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench_ref=$?
BENCH_NO_CPU=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_c2.json gpurun_out/bench_c1.json gpurun_out/bench_c3.json gpurun_out/bench_ref.json | cut -c1-600
