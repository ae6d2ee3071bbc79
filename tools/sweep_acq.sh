# developer: dependency-wait acquire variants (dev library) at n = 15, 16
export PTDR_LIB_NAME=libptdr_dev.so
run() { echo -n "$* : "; env "$@" timeout 200 python tools/diag_n15.py $N 2>&1 | tail -1; }
for rep in 1 2; do for N in 15 16; do export N
run PTDR_ACQ=0
run PTDR_ACQ=2
done; done
