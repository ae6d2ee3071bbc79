# developer: round-2 measurement set (one B200): bench line, reference arm, the bench
# command's ncu launch list, and one ncu --set full capture of the dense kernel
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.jsonl 2> gpurun_out/bench_r02.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02.jsonl
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.jsonl 2> gpurun_out/bench_ref_r02.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_small_r02.jsonl 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench_r02.log 2>&1
echo "ncu list rc=$?"
python tools/diag_n15.py 15 > gpurun_out/diag_plain_r02.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:dense_pipe_kernel -s 3 -c 1 \
    -o gpurun_out/prof_pipe_r02 python tools/diag_n15.py 15 > gpurun_out/prof_pipe_r02.log 2>&1
echo "ncu full rc=$?"
