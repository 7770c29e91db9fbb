#!/bin/bash
# round-2 GPU batch: new GPU tests, SpMM slab A/B on C4 and C2, full GPU suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/t_sharded.log 2>&1; echo "sharded rc=$?"
tail -3 gpurun_out/t_sharded.log
python -m pytest tests/test_gpu_parity.py -x -q -k "slab or variants" > gpurun_out/t_slab.log 2>&1; echo "slab rc=$?"
tail -3 gpurun_out/t_slab.log
timeout 1200 python tools/ab_spmm_slab.py c4 0,4096,20480,53248,86016,8192,24576 > gpurun_out/ab_slab_c4.log 2>&1; echo "ab c4 rc=$?"
cat gpurun_out/ab_slab_c4.log
timeout 600 python tools/ab_spmm_slab.py c2 0,4096,20480,53248,8192,24576 > gpurun_out/ab_slab_c2.log 2>&1; echo "ab c2 rc=$?"
cat gpurun_out/ab_slab_c2.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo "all rc=$?"
tail -5 gpurun_out/t_all.log
