#!/bin/bash
mkdir -p gpurun_out
python tools/inverse_layout_once.py 15 || exit 1
python tools/inverse_once.py 15
ncu --set full --clock-control none -k regex:dense_pipe_kernel -s 2 -c 1 -o gpurun_out/prof_inv_layout -f \
    python tools/inverse_layout_once.py 15 > /dev/null 2>&1
echo done
