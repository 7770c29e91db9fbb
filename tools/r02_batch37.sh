#!/bin/bash
# output prefault during the solve: host_io tests, GPU suite, C4 / C2 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_io.py -q -x > gpurun_out/hio37.log 2>&1; echo host_io_rc=$?; tail -3 gpurun_out/hio37.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gt37.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt37.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt37.log | head
for c in c4 c2; do
timeout 900 python bench.py --no-cpu-baseline --config $c > gpurun_out/b37_${c}.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/b37_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), 'pageable', d['e2e_pageable']['value'], d['clocks'])"
done
