#!/bin/bash
# HERMITIAN_TRIDIAGONAL: tests + n=24 timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tridiag_fused.py tests/test_gpu_generator.py -x -q -m gpu > gpurun_out/htri_tests.log 2>&1
echo "tests exit $?"; tail -15 gpurun_out/htri_tests.log
python tools/band_times.py 24 2>&1 | grep tridiag | cut -c1-160
