#!/bin/bash
# developer: band parity + n=24 timings + launch list of the current build
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band or zshard or n24 or max_n28 or tridiag or diagonal or guard" > gpurun_out/gpu_tests_band_ab.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_band_ab.log
python tools/band_times.py 24 > gpurun_out/band_times_ab.jsonl 2>&1; cat gpurun_out/band_times_ab.jsonl
python tools/band_once.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_ab.csv python tools/band_once.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_band_ab.csv | grep -v gen_band
