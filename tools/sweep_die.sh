# developer: die-aware split on/off (dev library) at n = 13..16, plus dense parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or configs or sharded or inplace or upper or guard or generated or peer or padded" > gpurun_out/gpu_tests_die.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_die.log
export PTDR_LIB_NAME=libptdr_dev.so
for rep in 1 2 3; do
for n in 15 16 14; do
  echo -n "n=$n die : "; timeout 200 python tools/diag_n15.py $n 2>&1 | tail -1
  echo -n "n=$n nodie : "; PTDR_NO_DIE=1 timeout 200 python tools/diag_n15.py $n 2>&1 | tail -1
done
done
