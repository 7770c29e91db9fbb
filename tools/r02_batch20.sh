# exchange overlap (panelled A^T pass): sharded + parity suites; C5 / C3 slab A/B through bench.py
python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/gt_sh.log 2>&1; echo sharded_rc=$?; tail -2 gpurun_out/gt_sh.log
python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined_variants or eig_overlap or loop_options" > gpurun_out/gt_par.log 2>&1; echo parity_rc=$?; tail -2 gpurun_out/gt_par.log
for o in 0 32 64; do
python bench.py --no-cpu-baseline --config c5 --steps 3 --option spmm_slab=$o > gpurun_out/b8_c5_$o.log 2>&1
tail -1 gpurun_out/b8_c5_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 slab $o', round(d['value']*1e3,2), 'ms', d['breakdown_last_step']['spmm_pass_ms'])"
done
