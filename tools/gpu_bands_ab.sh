#!/bin/bash
# developer: band(s) tests + timings + launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band_s or band or maxsize or guard" > gpurun_out/gpu_tests_bands.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_bands.log
python tools/band_s_once.py 24 2; python tools/band_s_once.py 22 5; python tools/band_s_once.py 20 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bands2.csv python tools/band_s_once.py 24 2 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bands2.csv | tail -6
