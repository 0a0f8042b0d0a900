#!/bin/bash
mkdir -p gpurun_out
python tools/variant_bench.py 2 20; python tools/variant_bench.py 4 10
HSIM_TRACE=1 python tools/trace_sweep.py 2 3 2> gpurun_out/trace8.log; grep -A40 "call 2" gpurun_out/trace8.log
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"6k_pipeILi4E" -s 1 -c 1 -o gpurun_out/prof8_pipe4 python tools/prof_sweep.py 2 2 > gpurun_out/ncu8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"k_final_small" -s 1 -c 1 -o gpurun_out/prof8_final python tools/prof_sweep.py 2 2 >> gpurun_out/ncu8.log 2>&1
tail -3 gpurun_out/ncu8.log; ls gpurun_out/*.ncu-rep
