# developer: dense n=15 scratch-ring / discard / look-ahead sweep on the dev library
export PTDR_LIB_NAME=libptdr_dev.so
run() { echo -n "$* : "; env "$@" timeout 120 python tools/diag_n15.py 15 2>&1 | tail -1; }
for rep in 1 2; do
run PTDR_X=default
run PTDR_NSLOT=4 PTDR_NO_DISCARD=1
run PTDR_NSLOT=8 PTDR_NO_DISCARD=1
run PTDR_NSLOT=4
run PTDR_NSLOT=8
run PTDR_NSLOT=16 PTDR_NO_DISCARD=1
run PTDR_NSLOT=8 PTDR_NO_DISCARD=1 PTDR_L=3
run PTDR_NSLOT=8 PTDR_L=3
done
