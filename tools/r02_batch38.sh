#!/bin/bash
# host copy micro on the GPU box's host, then C4 / C2 bench with the streaming host copy
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|^CPU\(s\)"
/usr/bin/g++-13 -O2 -fopenmp -std=c++17 paper_2404_09276_b200/csrc/host_io.cpp tools/micro/host_copy.cpp -o /tmp/host_copy && timeout 300 /tmp/host_copy | tee gpurun_out/host_copy38.txt
timeout 600 python -m pytest tests/test_gpu_host_io.py -q -x > gpurun_out/hio38.log 2>&1; echo host_io_rc=$?; tail -1 gpurun_out/hio38.log
for c in c4 c2; do
timeout 900 python bench.py --no-cpu-baseline --config $c > gpurun_out/b38_${c}.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/b38_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), 'pageable', d['e2e_pageable']['value'], d['clocks'])"
done
for t in 8 4; do
timeout 900 python bench.py --no-cpu-baseline --config c4 --steps 3 --option host_copy_threads=$t > gpurun_out/b38_c4_t$t.log 2>&1
tail -1 gpurun_out/b38_c4_t$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 threads $t e2e', round(d['e2e']['value']*1e3,2), 'pageable', d['e2e_pageable']['value'])"
done
