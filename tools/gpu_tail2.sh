#!/bin/bash
# developer: fine-grained tail groups -- band parity, timings, look sweep (dev library), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band or zshard or n24 or max_n28 or tridiag or diagonal or guard" > gpurun_out/gpu_tests_tail2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_tail2.log
python tools/band_times.py 24 > gpurun_out/band_times_tail2.jsonl 2>&1; cat gpurun_out/band_times_tail2.jsonl
export PTDR_LIB_NAME=libptdr_dev.so
for look in 1 2 4 8 16 32; do echo "look=$look"; PTDR_TAIL_LOOK=$look python tools/band_times.py 24 2>&1 | grep '"world": 1,\|"world": 8,'; done
unset PTDR_LIB_NAME
python tools/band_once.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_tail2.csv python tools/band_once.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_band_tail2.csv | grep -v gen_band
