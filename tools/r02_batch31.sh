#!/bin/bash
# final verification of the round-2 build: product GPU suite, the bounds-checked build's GPU
# suite, smoke(), and a C4 launch list with DRAM bytes (v4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_final.log 2>&1; echo "product rc=$?"; tail -1 gpurun_out/t_final.log
DSVD_CHECKED=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_final_checked.log 2>&1; echo "checked rc=$?"; tail -1 gpurun_out/t_final_checked.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_launches_c4_v4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_c4_v4.log 2>&1; echo "launch list rc=$?"
