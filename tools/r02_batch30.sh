# after the fused exchange (both halves): GPU suite + C4 bench line
python -m pytest tests -m gpu -q > gpurun_out/gt15.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt15.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt15.log | head
python bench.py --no-cpu-baseline > gpurun_out/b16_c4.log 2>&1
tail -1 gpurun_out/b16_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), d['breakdown_last_step'])"
