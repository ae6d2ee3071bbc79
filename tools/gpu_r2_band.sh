# developer: z-shard / band tests, band timings and the die hand-off microbenchmark (one B200)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_bench tools/die_bench.cu
timeout 600 ./tools/die_bench > gpurun_out/die_bench.txt 2>&1; echo "die_bench rc=$?"; cat gpurun_out/die_bench.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "zshard or band or sharded or inplace or n24 or max_n28" > gpurun_out/gpu_tests_band.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests_band.log
timeout 600 python tools/band_times.py 24 > gpurun_out/band_times.jsonl 2>&1; echo "band_times rc=$?"; cat gpurun_out/band_times.jsonl
