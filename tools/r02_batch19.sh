# column-slab kernel at l = 150 on the big configs (C5, C3): A/B of spmm_slab
python tools/ab_option.py c5 spmm_slab 0,64,32 --no-bench > gpurun_out/ab_slab_c5.log 2>&1; tail -3 gpurun_out/ab_slab_c5.log
python tools/ab_option.py c3 spmm_slab 0,64,32 --no-bench > gpurun_out/ab_slab_c3.log 2>&1; tail -3 gpurun_out/ab_slab_c3.log
