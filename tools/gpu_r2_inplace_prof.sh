mkdir -p gpurun_out
python tools/inplace_once.py 15 > gpurun_out/ip_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:dense_pipe_kernel -s 3 -c 1 -o gpurun_out/prof_inplace_r02 python tools/inplace_once.py 15 > gpurun_out/prof_inplace_r02.log 2>&1
echo "ncu rc=$?"
