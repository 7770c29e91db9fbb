#!/bin/bash
# C4: launch list of a short bench run and a full ncu capture of the SpMM (slab) kernels of a p=1 solve
cd "$(dirname "$0")/.."
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_c4.log 2>&1; echo "launch list rc=$?"
timeout 1200 $NCU --set full --clock-control none -k regex:"spmm_slab|split_combine|empty_rows" -c 8 -o gpurun_out/c4_slab3 -f \
    python tools/ncu_spmm.py c4 solve > gpurun_out/ncu_c4_slab3.log 2>&1; echo "ncu rc=$?"
