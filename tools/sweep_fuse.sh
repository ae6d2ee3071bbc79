#!/bin/bash
export PTDR_LIB_NAME=libptdr_dev.so
for m in 7 5 4 3 2; do echo "maxt(KS=1)=$m"; PTDR_FUSE_MAXT1=$m python tools/band_times.py 24 2>&1 | grep '"world": 8' | grep tridiag | cut -c1-120; done
