#!/bin/bash
# C5 on the final build: reference-free self-check at full scale (R-MAT 24) and the
# C5-shaped parity against the unmodified reference at R-MAT scale 23
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/self_check_large.py c5 > gpurun_out/selfcheck_c5.log 2>&1; echo "selfcheck rc=$?"; tail -2 gpurun_out/selfcheck_c5.log
timeout 2400 python tools/parity_large.py c5 --rmat-scale 23 > gpurun_out/parity_c5_s23.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/parity_c5_s23.log
