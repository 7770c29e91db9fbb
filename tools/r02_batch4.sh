#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "slab" > gpurun_out/t_slab2.log 2>&1; echo "slab tests rc=$?"; tail -2 gpurun_out/t_slab2.log
timeout 900 python tools/ab_option.py c4 spmm_slab 0,32,64 > gpurun_out/ab_c4_slab_layout.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_c4_slab_layout.log
timeout 900 python tools/ab_option.py c4 slab_layout 0,1 spmm_slab=64 > gpurun_out/ab_c4_layout01.log 2>&1; cat gpurun_out/ab_c4_layout01.log
timeout 600 python tools/ab_option.py c2 spmm_slab 0,32,64 > gpurun_out/ab_c2_slab_layout.log 2>&1; cat gpurun_out/ab_c2_slab_layout.log
