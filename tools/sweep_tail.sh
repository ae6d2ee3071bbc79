# developer: tail-pipeline look-ahead (dev library), n = 24 diagonal / tridiagonal, 1 GPU
export PTDR_LIB_NAME=libptdr_dev.so
for look in 0 1 2 3; do echo "look=$look"; PTDR_TAIL_LOOK=$look python tools/band_times.py 24 2>&1 | grep '"world": 1,'; done
