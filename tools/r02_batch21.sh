# defaults after the exchange overlap / slab-32 rule: GPU suite + bench lines of every config
python -m pytest tests -m gpu -x -q > gpurun_out/gt5.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt5.log
for c in c5 c3 c2 c4; do
python bench.py --no-cpu-baseline --config $c > gpurun_out/b9_${c}.log 2>&1
tail -1 gpurun_out/b9_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), d['breakdown_last_step'])"
done
