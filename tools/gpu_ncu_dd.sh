set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_split|k_final" -s 2 -c 2 -o gpurun_out/prof_dd_split_final python tools/prof_sweep.py 2 2 > gpurun_out/ncu_dd.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_dd.csv python tools/prof_sweep.py 2 2 > /dev/null 2>&1
ls -la gpurun_out
