#!/bin/bash
# One GPU call: bench line, ncu launch list of one sweep, one full ncu capture of
# the dominant kernel (K_pipe<4>), then summaries under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_sweep.py 2 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 0 -c 1 -o gpurun_out/prof_pipe4 python tools/prof_sweep.py 2 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"k_split|k_sync|k_deep|k_final" -s 0 -c 4 -o gpurun_out/prof_phases python tools/prof_sweep.py 2 1 >> gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bench.json gpurun_out/bench_ref.json
