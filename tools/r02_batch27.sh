# whole-row short rows (default): GPU suite, A/B on C5 / C3 (32-column slabs), C4 bench line
python -m pytest tests -m gpu -q > gpurun_out/gt10.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt10.log; grep -E '^(FAILED|ERROR)' gpurun_out/gt10.log | head
for c in c5 c3; do for o in 0 1; do
python bench.py --no-cpu-baseline --config $c --steps 3 --option spmm_short_rows=$o > gpurun_out/b13_${c}_$o.log 2>&1
tail -1 gpurun_out/b13_${c}_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c short=$o', round(d['value']*1e3,2), 'ms', d['breakdown_last_step']['spmm_pass_ms'])"
done; done
python bench.py --no-cpu-baseline > gpurun_out/b13_c4.log 2>&1
tail -1 gpurun_out/b13_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value']*1e3,2), 'ms e2e', round(d['e2e']['value']*1e3,2), d['breakdown_last_step'])"
