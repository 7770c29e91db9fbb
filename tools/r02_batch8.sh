#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -x -q -k "slab" > gpurun_out/t_slab5.log 2>&1; echo "slab tests rc=$?"; tail -2 gpurun_out/t_slab5.log
timeout 900 python tools/ab_option.py c4 spmm_hot_mb 0,48,96,160 spmm_slab=64,spmm_slab_depth=2 > gpurun_out/ab_c4_hot64.log 2>&1; cat gpurun_out/ab_c4_hot64.log
timeout 900 python tools/ab_option.py c4 spmm_hot_mb 0,96,160 spmm_slab=32,spmm_slab_depth=2 > gpurun_out/ab_c4_hot32.log 2>&1; cat gpurun_out/ab_c4_hot32.log
