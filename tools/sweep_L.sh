# developer: look-ahead sweep (dev library) with the current pipeline
export PTDR_LIB_NAME=libptdr_dev.so
run() { echo -n "$* : "; env "$@" timeout 200 python tools/diag_n15.py $N 2>&1 | tail -1; }
for rep in 1 2; do
N=16; export N; run PTDR_L=1; run PTDR_L=2; run PTDR_L=3
N=15; export N; run PTDR_L=2; run PTDR_L=3; run PTDR_L=4
N=14; export N; run PTDR_L=3; run PTDR_L=5; run PTDR_L=8
done
