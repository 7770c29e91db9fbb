#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -k "slab or sharded or spmm" > gpurun_out/t_b9.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_b9.log
timeout 900 python tools/ab_option.py c4 spmm_slab 0,64 > gpurun_out/ab_c4_b9.log 2>&1; cat gpurun_out/ab_c4_b9.log
