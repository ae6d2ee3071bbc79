#!/bin/bash
# developer: ncu --set full of the q-order inverse (MODE_INVQ) and the matrix-layout inverse at n = 15
mkdir -p gpurun_out
python tools/inverse_once.py 15 > gpurun_out/invq_once.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:dense_pipe_kernel -s 2 -c 1 -o gpurun_out/prof_invq -f \
    python tools/inverse_once.py 15 > gpurun_out/prof_invq.log 2>&1
echo done
