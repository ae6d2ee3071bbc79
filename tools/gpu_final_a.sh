#!/bin/bash
# round-2 refresh: full GPU suite, smoke, bench, configs (incl. next rows), n=24 band timings
bash tools/gpu_suite.sh
timeout 900 python tools/tools_bench_configs.py all > gpurun_out/configs_r02c.jsonl 2> gpurun_out/configs_r02c.err; echo "configs rc=$?"
python tools/band_times.py 24 > gpurun_out/band_times_r02c.jsonl 2>&1
cat gpurun_out/configs_r02c.jsonl | cut -c1-200
