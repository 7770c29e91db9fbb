#!/bin/bash
# last session of round 2, on the tree rebuilt from a fresh container: C4 launch list with DRAM
# bytes (v5), the other configs' bench lines, then full-size C4 parity (p = 30) against the
# unmodified reference (~32 min on 16 cores)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/s4_bench_$c.json 2> gpurun_out/s4_bench_$c.err; echo "bench $c rc=$?"; cut -c1-120 gpurun_out/s4_bench_$c.json
done
timeout 1500 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_launches_c4_v5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_c4_v5.log 2>&1; echo "launch list rc=$?"
timeout 3000 python tools/parity_large.py c4 > gpurun_out/parity_c4_s4.log 2>&1; echo "c4 parity rc=$?"; tail -1 gpurun_out/parity_c4_s4.log | cut -c1-600
