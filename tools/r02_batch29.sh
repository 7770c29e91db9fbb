# eig_overlap 3 (short eig kernels at default priority beside the A T pass): tests + C2 / C4 A/B
python -m pytest tests/test_gpu_parity.py -q -k "eig_overlap or pipelined_variants or loop_options" > gpurun_out/gt12.log 2>&1; echo rc=$?; tail -2 gpurun_out/gt12.log
for c in c2 c4; do for o in -1 3; do
python bench.py --no-cpu-baseline --config $c --option eig_overlap=$o > gpurun_out/b15_${c}_$o.log 2>&1
tail -1 gpurun_out/b15_${c}_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c eov=$o', round(d['value']*1e3,2), 'ms', d['breakdown_last_step']['spmm_pass_ms'])"
done; done
