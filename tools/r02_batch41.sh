#!/bin/bash
# final tree: the bounds-checked build's GPU suite, then C5-shaped parity at R-MAT 23 against the
# unmodified reference (~14 min on 16 cores)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DSVD_CHECKED=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_suite_checked.log 2>&1; echo "checked rc=$?"; tail -1 gpurun_out/s4_suite_checked.log
timeout 1800 python tools/parity_large.py c5 --rmat-scale 23 > gpurun_out/parity_c5_s4.log 2>&1; echo "c5 parity rc=$?"; tail -1 gpurun_out/parity_c5_s4.log | cut -c1-700
