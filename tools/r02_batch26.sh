#!/bin/bash
# final round-2 bench lines: the driver-equivalent default run (C4, with the reference's bounded
# sample as cpu_baseline) and every other config on this build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4_final.json 2> gpurun_out/r02_bench_c4_final.err; echo "c4 rc=$?"
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_${c}_final.json 2> gpurun_out/r02_bench_${c}_final.err
  echo "$c rc=$?"
done
for c in c4 c1 c2 c3 c5; do python -c "import json;d=json.load(open('gpurun_out/r02_bench_${c}_final.json'));print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"; done
