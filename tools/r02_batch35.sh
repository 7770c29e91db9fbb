#!/bin/bash
# post-compaction re-sweep of the dense-kernel grid knobs and the slab SpMM knobs on C4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "gram_waves 24,16,32,48" "rescale_row_ctas 4096,2048,8192,16384" "spmm_slab_depth 2,1" "spmm_slab_hint 2,0,1"; do
  set -- $spec
  timeout 600 python tools/ab_option.py c4 $1 $2 --no-bench 2>&1 | grep -v Warning
done > gpurun_out/ab35.log
cat gpurun_out/ab35.log
