#!/bin/bash
# developer: tridiagonal P/M chain -- parity, timings (product), A/B and look sweep (dev library)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band or zshard or n24 or max_n28 or tridiag or diagonal or guard" > gpurun_out/gpu_tests_chain.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_chain.log
python tools/band_times.py 24 2>&1 | grep tridiag
export PTDR_LIB_NAME=libptdr_dev.so
echo nochain; PTDR_TRI_NOCHAIN=1 python tools/band_times.py 24 2>&1 | grep tridiag
for look in 0 1 2 4; do echo "look=$look"; PTDR_CHAIN_LOOK=$look python tools/band_times.py 24 2>&1 | grep tridiag; done
unset PTDR_LIB_NAME
python tools/band_once.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_chain.csv python tools/band_once.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_band_chain.csv | grep -v gen_band | tail -16
