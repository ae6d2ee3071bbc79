#!/bin/bash
mkdir -p gpurun_out
python tools/gen_once.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:dense_pipe_kernel -s 1 -c 1 -o gpurun_out/prof_gen -f python tools/gen_once.py > /dev/null 2>&1
ncu --set full --clock-control none -k regex:gen_dense -s 1 -c 1 -o gpurun_out/prof_gendense -f python tools/gen_once.py > /dev/null 2>&1
echo done
