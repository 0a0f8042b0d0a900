set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_gputest.log 2>&1; tail -2 gpurun_out/fin_gputest.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; cat gpurun_out/fin_bench.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/fin_bench_ref.json 2>&1; tail -1 gpurun_out/fin_bench_ref.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_sweep.py 2 2 > /dev/null 2>&1
