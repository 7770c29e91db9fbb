#!/bin/bash
# A/B of the 2x2-tile wide Gram's k-step unroll (2 = product, 4, 8) on C4: variant libraries built
# into tools/_var/uN (dmma.cu with -DDSVD_GW2_UNROLL=N), swapped in on the box's scratch copy
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2404_09276_b200/_lib/libdashsvd_b200.so /tmp/lib_u2.so
for v in u2 u4 u8 u2; do
  if [ $v = u2 ]; then cp /tmp/lib_u2.so paper_2404_09276_b200/_lib/libdashsvd_b200.so; else cp tools/_var/$v/libdashsvd_b200.so paper_2404_09276_b200/_lib/libdashsvd_b200.so; fi
  timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ab_gw2_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_gw2_$v.json').read().strip().splitlines()[-1]); b=d['breakdown_last_step']
print('$v', 'solve', round(d['value'],4), 'gram_ms', b['gram_ms'], 'rescale_ms', b['rescale_ms'], 'spmm_ms', b['spmm_ms'])" | tee -a gpurun_out/ab_gw2_unroll.txt
done
cp /tmp/lib_u2.so paper_2404_09276_b200/_lib/libdashsvd_b200.so
