#!/bin/bash
cd "$(dirname "$0")/.."
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none -k regex:"spmm_slab|slab_copy" -c 6 -o gpurun_out/c4_slab2 -f \
    python tools/ncu_spmm.py c4 solve spmm_slab=64 spmm_slab_depth=2 spmm_slab_pf=0 > gpurun_out/ncu_c4_slab2.log 2>&1; echo "ncu rc=$?"
