mkdir -p gpurun_out
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 3 2 > gpurun_out/r2h_trace_def.log 2>&1
HSIM_LIB=paper_2508_05370_b200/variants/libhsim_mm0.so HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 3 2 > gpurun_out/r2h_trace_mm0.log 2>&1
