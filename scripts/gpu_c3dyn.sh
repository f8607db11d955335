#!/bin/bash
# C3 A/B: RoPE trees in the split-K QKV epilogue (last split / cooperative) vs the separate eltwise
mkdir -p gpurun_out
VTC_TREE_COOP=1 timeout 900 python -m pytest tests/test_decode_steps.py tests/test_fullsize.py -q -x -m gpu -k "dynamic or c3" -s > gpurun_out/c3d_tests.log 2>&1; echo tests=$?; grep -E "rel err|passed|failed|Error" gpurun_out/c3d_tests.log | tail -8
export BENCH_NO_CPU=1
run() { timeout 600 env "$@" python bench.py --config c3 --steps 20 > gpurun_out/c3d.json 2> gpurun_out/c3d.err; echo "$@" rc=$?
python -c "import json; d=json.load(open('gpurun_out/c3d.json')); print(round(d['value'],1), [(l['node'][:12],round(l['us'],1)) for l in d['launch_timeline']])"; }
run X=1
run VTC_TREE_COOP=1
run VTC_NO_TC_TREES=1
run VTC_TREE_COOP=1
