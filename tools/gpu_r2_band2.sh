# developer: z-shard / band parity + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "zshard or band or n24 or max_n28 or antidiag or tridiag or diagonal" > gpurun_out/gpu_tests_band2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_band2.log
timeout 600 python tools/band_times.py 24 > gpurun_out/band_times2.jsonl 2>&1; echo "band_times rc=$?"; cat gpurun_out/band_times2.jsonl
python tools/band_once.py > gpurun_out/band_once_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_r2b.csv python tools/band_once.py > gpurun_out/band_once_ncu.log 2>&1
echo "ncu rc=$?"
