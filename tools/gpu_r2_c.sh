# developer: die hand-off v2 + band parity/timings
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_bench tools/die_bench.cu
timeout 600 ./tools/die_bench > gpurun_out/die_bench2.txt 2>&1; echo "die_bench rc=$?"; cat gpurun_out/die_bench2.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "zshard or n24 or max_n28" > gpurun_out/gpu_tests_band3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_band3.log
timeout 600 python tools/band_times.py 24 > gpurun_out/band_times3.jsonl 2>&1; echo "band_times rc=$?"; cat gpurun_out/band_times3.jsonl
