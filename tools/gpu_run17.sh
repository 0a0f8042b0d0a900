#!/bin/bash
mkdir -p gpurun_out
CONFIGS="2 4 3" bash tools/variants_run.sh fp6 fp4 fp1 deepfirst nb2 > gpurun_out/variants17.log 2>&1; cat gpurun_out/variants17.log
HSIM_TRACE=1 python tools/trace_sweep.py 2 3 2> gpurun_out/trace17.log; grep -A30 "call 2" gpurun_out/trace17.log
