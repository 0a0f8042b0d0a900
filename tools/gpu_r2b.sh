set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2b.log 2>&1; tail -3 gpurun_out/gputest_r2b.log
timeout 300 python tools/e2e_chunks.py > gpurun_out/e2e_chunks.log 2>&1; cat gpurun_out/e2e_chunks.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; cat gpurun_out/bench_r2b.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_sweep.py 2 2 > /dev/null 2>&1
