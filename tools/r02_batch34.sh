#!/bin/bash
# re-entry check of the final build: GPU suite, smoke, default bench (C4, no CPU leg)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gt34.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt34.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt34.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke34.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke34.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b34_c4.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/b34_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), d['clocks'], d['breakdown_last_step'])"
