#!/bin/bash
# ncu of the column-slab SpMM kernels on C4 (32- and 64-column slabs, both passes)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --set full --clock-control none -k regex:"spmm_slab" -c 8 -o gpurun_out/c4_slab -f \
    python tools/ncu_spmm.py c4 spmm 4096,8192 > gpurun_out/ncu_c4_slab.log 2>&1; echo "ncu slab rc=$?"
