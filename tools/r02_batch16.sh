#!/bin/bash
# round-2 late: full GPU suite, then bench lines for every config with the current build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all16.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/t_all16.log
for c in c2 c3 c5 c1; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench16_$c.json 2> gpurun_out/bench16_$c.err
  echo "$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench16_$c.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_last_step'])"
done
