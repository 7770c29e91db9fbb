#!/bin/bash
# ncu captures on C4: SpMM (whole-row vs 32/64-column slabs) and the dense kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/t_sharded.log 2>&1; echo "sharded rc=$?"; tail -2 gpurun_out/t_sharded.log
timeout 1500 $NCU --set full --clock-control none -k regex:"spmm_(slab|row)" -c 6 -o gpurun_out/c4_spmm -f \
    python tools/ncu_spmm.py c4 spmm 0,4096,8192 > gpurun_out/ncu_c4_spmm.log 2>&1; echo "ncu spmm rc=$?"
timeout 900 $NCU --set full --clock-control none -k regex:"gram_dmma_wide|rescale_tma" -c 3 -o gpurun_out/c4_dense -f \
    python tools/ncu_spmm.py c4 solve > gpurun_out/ncu_c4_dense.log 2>&1; echo "ncu dense rc=$?"
tail -3 gpurun_out/ncu_c4_spmm.log gpurun_out/ncu_c4_dense.log
