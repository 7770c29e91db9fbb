#!/bin/bash
# full-size parity on the final build: C4 at p = 30 (reference ~32 min on 16 cores), C5-shaped at R-MAT 23
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSVD_BUILD=58d299e
timeout 3000 python tools/parity_large.py c4 > gpurun_out/parity_c4_final.log 2>&1; echo "c4 parity rc=$?"; tail -1 gpurun_out/parity_c4_final.log | cut -c1-600
timeout 1500 python tools/parity_large.py c5 --rmat-scale 23 > gpurun_out/parity_c5_final.log 2>&1; echo "c5 parity rc=$?"; tail -1 gpurun_out/parity_c5_final.log | cut -c1-600
