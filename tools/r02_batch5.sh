#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -x -q -k "slab" > gpurun_out/t_slab3.log 2>&1; echo "slab tests rc=$?"; tail -2 gpurun_out/t_slab3.log
timeout 900 python tools/ab_option.py c4 spmm_slab_pf 0,1 spmm_slab=64 > gpurun_out/ab_c4_pf64.log 2>&1; cat gpurun_out/ab_c4_pf64.log
timeout 900 python tools/ab_option.py c4 spmm_slab_pf 0,1 spmm_slab=32 > gpurun_out/ab_c4_pf32.log 2>&1; cat gpurun_out/ab_c4_pf32.log
timeout 900 python tools/ab_option.py c4 spmm_slab_depth 1,2 spmm_slab=32,spmm_slab_pf=1 > gpurun_out/ab_c4_depth.log 2>&1; cat gpurun_out/ab_c4_depth.log
timeout 600 python tools/ab_option.py c2 spmm_slab 0,32,64 > gpurun_out/ab_c2_pf.log 2>&1; cat gpurun_out/ab_c2_pf.log
