#!/bin/bash
# developer: every band / tridiagonal GPU test + n=24 timings
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band or zshard or n24 or max_n28 or tridiag or diagonal or guard or generator" > gpurun_out/gpu_tests_bandfull.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_bandfull.log
python tools/band_times.py 24 2>&1 | cut -c1-150
