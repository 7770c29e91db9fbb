#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -x -q -k "slab" > gpurun_out/t_slab4.log 2>&1; echo "slab tests rc=$?"; tail -2 gpurun_out/t_slab4.log
timeout 900 python tools/ab_option.py c4 spmm_slab_depth 0,1,2 spmm_slab=64,spmm_slab_pf=0 > gpurun_out/ab_c4_d64.log 2>&1; cat gpurun_out/ab_c4_d64.log
timeout 900 python tools/ab_option.py c4 spmm_slab_depth 0,1,2 spmm_slab=32,spmm_slab_pf=0 > gpurun_out/ab_c4_d32.log 2>&1; cat gpurun_out/ab_c4_d32.log
timeout 600 python tools/ab_option.py c2 spmm_slab_depth 0,1 spmm_slab=32,spmm_slab_pf=0 > gpurun_out/ab_c2_d32.log 2>&1; cat gpurun_out/ab_c2_d32.log
