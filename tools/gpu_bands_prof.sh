#!/bin/bash
# developer: band(s) n=24 s=2 / n=22 s=5 launch lists
mkdir -p gpurun_out
python tools/band_s_once.py 24 2 > gpurun_out/bands_once.log 2>&1 || exit 1
cat gpurun_out/bands_once.log
python tools/band_s_once.py 22 5 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bands.csv python tools/band_s_once.py 24 2 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bands.csv | tail -12
