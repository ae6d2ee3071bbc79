# developer: dense parity subset + n=15/16 timing (product library) + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or configs or sharded or inplace or upper or generated or peer or padded or guard" > gpurun_out/gpu_tests_dense.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_dense.log
for rep in 1 2 3; do for n in 15 16 13; do echo -n "n=$n "; timeout 200 python tools/diag_n15.py $n 2>&1 | tail -1; done; done
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1
