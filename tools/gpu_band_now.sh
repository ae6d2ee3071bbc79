#!/bin/bash
# developer: n=24 structured timings + launch list of the current build
mkdir -p gpurun_out
python tools/band_times.py > gpurun_out/band_now.jsonl 2> gpurun_out/band_now.err || exit 1
python tools/band_once.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_now.csv python tools/band_once.py > /dev/null 2>&1
cat gpurun_out/band_now.jsonl
python tools/launch_summary.py gpurun_out/launches_band_now.csv
