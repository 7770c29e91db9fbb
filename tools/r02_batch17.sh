python -m pytest tests -m gpu -x -q > gpurun_out/gt3.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/gt3.log
for c in c4 c2; do for o in 2 1; do
python bench.py --no-cpu-baseline --config $c --option eig_overlap=$o > gpurun_out/b6_${c}_${o}.log 2>&1
tail -1 gpurun_out/b6_${c}_${o}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'eig_overlap=$o', round(d['value']*1e3,2), 'ms', 'e2e', round(d['e2e']['value']*1e3,2), d['breakdown_last_step']['spmm_pass_ms'])"
done; done
