#!/bin/bash
# q-order inverse on the pipeline: tests + timings
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_algebra.py tests/test_gpu_inverse_layout.py tests/test_gpu_guard.py -x -q -m gpu > gpurun_out/invq_tests.log 2>&1
echo "tests exit $?"; tail -3 gpurun_out/invq_tests.log
timeout 600 python tools/tools_bench_configs.py inverse > gpurun_out/invq_times.jsonl 2> gpurun_out/invq_times.err
cat gpurun_out/invq_times.jsonl | cut -c1-250
