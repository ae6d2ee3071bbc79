#!/bin/bash
# round-2 refresh B: full GPU suite, smoke, bench, configs, n=24 band timings, band(s) timings
bash tools/gpu_suite.sh
timeout 900 python tools/tools_bench_configs.py all > gpurun_out/configs_r02d.jsonl 2> gpurun_out/configs_r02d.err; echo "configs rc=$?"
python tools/band_times.py 24 > gpurun_out/band_times_r02d.jsonl 2>&1
cat gpurun_out/configs_r02d.jsonl | cut -c1-160
