set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dedup_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/dd3_test.log 2>&1; tail -3 gpurun_out/dd3_test.log
for c in 2 4 3; do timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/dd3_var.log 2>&1; done
cat gpurun_out/dd3_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/dd3_trace.log 2>&1; tail -17 gpurun_out/dd3_trace.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_dd3.csv python tools/prof_sweep.py 2 2 > /dev/null 2>&1
