# row compaction in the finalize: GPU suite + C4 / C5 bench lines
python -m pytest tests -m gpu -q > gpurun_out/gt16.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt16.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt16.log | head
for c in c4 c5; do
python bench.py --no-cpu-baseline --config $c > gpurun_out/b17_${c}.log 2>&1
tail -1 gpurun_out/b17_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), d['breakdown_last_step'])"
done
