#!/bin/bash
# staged pageable host copies: new tests, GPU suite, C4 / C2 bench lines with e2e_pageable
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_io.py -q -x > gpurun_out/hio36.log 2>&1; echo host_io_rc=$?; tail -15 gpurun_out/hio36.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gt36.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt36.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt36.log | head
for c in c4 c2; do
timeout 900 python bench.py --no-cpu-baseline --config $c > gpurun_out/b36_${c}.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/b36_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), 'pageable', d['e2e_pageable'], d['clocks'])"
done
for c in c2 c4; do
timeout 900 python bench.py --no-cpu-baseline --config $c --option host_staging=0 > gpurun_out/b36_${c}_nostage.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/b36_${c}_nostage.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c host_staging=0', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), 'pageable', d['e2e_pageable'])"
done
