#!/bin/bash
# developer: ncu --set full of the first tail_pipe_kernel and seg_pass_kernel of tools/band_once.py
mkdir -p gpurun_out
python tools/band_once.py > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tail_pipe_kernel -c 1 -o gpurun_out/prof_tail -f \
    python tools/band_once.py > gpurun_out/prof_tail.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seg_pass_kernel -c 1 -o gpurun_out/prof_seg -f \
    python tools/band_once.py > gpurun_out/prof_seg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topk_pass_kernel -c 1 -o gpurun_out/prof_topk -f \
    python tools/band_once.py > gpurun_out/prof_topk.log 2>&1
echo done
