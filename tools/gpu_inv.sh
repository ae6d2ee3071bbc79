#!/bin/bash
# inverse transform from the matrix layout: tests + timings
set -o pipefail
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/inv_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_inverse_layout.py tests/test_gpu_inplace.py tests/test_gpu_algebra.py -x -q -m gpu > gpurun_out/inv_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/inv_tests.log
timeout 600 python tools/tools_bench_configs.py inverse > gpurun_out/inv_times.jsonl 2> gpurun_out/inv_times.err
tail -3 gpurun_out/inv_tests.log; cat gpurun_out/inv_times.jsonl
