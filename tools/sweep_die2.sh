# developer: producer registers 40, die split on/off, look-ahead, acquire fence (dev library)
mkdir -p gpurun_out
export PTDR_LIB_NAME=libptdr_dev.so
run() { echo -n "$* : "; env "$@" timeout 200 python tools/diag_n15.py $N 2>&1 | tail -1; }
for rep in 1 2; do
for N in 15 16; do
export N
run PTDR_NO_DIE=1
run PTDR_NO_DIE=1 PTDR_NO_ACQ=1
run PTDR_L=1
run PTDR_L=2
run PTDR_NO_DIE=1 PTDR_L=3
done
done
