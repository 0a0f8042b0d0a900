#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"k_split" -s 1 -c 1 -o gpurun_out/prof21_split python tools/prof_sweep.py 2 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"k_final_small" -s 1 -c 1 -o gpurun_out/prof21_final python tools/prof_sweep.py 2 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"6k_pipeILi4E" -s 1 -c 1 -o gpurun_out/prof21_pipe4 python tools/prof_sweep.py 2 2 > /dev/null 2>&1
ls -la gpurun_out/prof21*
