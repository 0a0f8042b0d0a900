#!/bin/bash
# launch-bound variants A/B + source-level ncu of K_sync and K_pipe<4>
mkdir -p gpurun_out
CONFIGS="2 4" bash tools/variants_run.sh pm6 pm5 s5 s4 p6s5 sp5 > gpurun_out/variants7.log 2>&1; cat gpurun_out/variants7.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_sync" -s 1 -c 1 -o gpurun_out/prof7_sync python tools/prof_sweep.py 2 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_pipe<4>" --kernel-name-base demangled -s 1 -c 1 -o gpurun_out/prof7_pipe4 python tools/prof_sweep.py 2 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_split" --kernel-name-base demangled -s 1 -c 1 -o gpurun_out/prof7_split python tools/prof_sweep.py 2 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
