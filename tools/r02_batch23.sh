#!/bin/bash
# C4 after column compaction + eig split: launch list with DRAM bytes of a short bench run,
# full ncu captures of the main slab SpMM launches, the rescale and the Gram of a solve
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_launches_c4_v3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_c4_v3.log 2>&1; echo "launch list rc=$?"
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"spmm_slab_kernel|rescale_tma|gram_dmma_wide2" \
    -c 10 -o gpurun_out/c4_v3 -f python tools/ncu_spmm.py c4 solve > gpurun_out/ncu_c4_v3.log 2>&1; echo "ncu rc=$?"
