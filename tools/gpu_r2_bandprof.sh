# developer: launch list (time + DRAM bytes) of the n=24 structured paths
mkdir -p gpurun_out
python tools/band_once.py > gpurun_out/band_once_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_band_r2.csv python tools/band_once.py > gpurun_out/band_once_ncu.log 2>&1
echo "rc=$?"
