set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_v4.log 2>&1; tail -3 gpurun_out/pytest_gpu_v4.log
python bench.py > gpurun_out/bench_v4.jsonl 2> gpurun_out/bench_v4.err; tail -1 gpurun_out/bench_v4.jsonl
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v4.jsonl 2> gpurun_out/bench_ref_v4.err; tail -1 gpurun_out/bench_ref_v4.jsonl
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench_v4.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench_v4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dense_pipe_kernel -s 3 -c 1 -o gpurun_out/prof_pipe_v4 python tools/diag_n15.py 15 > gpurun_out/prof_pipe_v4.log 2>&1
ls -la gpurun_out
