# developer: band parity + timings + launch list after the L2 tail pipeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "band or zshard or n24 or max_n28 or tridiag or diagonal or guard" > gpurun_out/gpu_tests_tail.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_tail.log
python tools/band_times.py 24 > gpurun_out/band_times_tail.jsonl 2>&1; cat gpurun_out/band_times_tail.jsonl
python tools/band_once.py > gpurun_out/band_once_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_tail.csv python tools/band_once.py > gpurun_out/band_once_ncu.log 2>&1
echo "ncu rc=$?"
