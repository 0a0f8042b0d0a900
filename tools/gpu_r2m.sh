mkdir -p gpurun_out
HSIM_LIB=paper_2508_05370_b200/variants/libhsim_seed.so timeout 120 python tools/seed_diag.py 2 > gpurun_out/r2m_seed.log 2>&1
HSIM_LIB=paper_2508_05370_b200/variants/libhsim_seed.so timeout 120 python tools/seed_diag.py 4 >> gpurun_out/r2m_seed.log 2>&1
cat gpurun_out/r2m_seed.log
HSIM_SEED=20228000000 HSIM_LIB=paper_2508_05370_b200/variants/libhsim_seed.so HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2m_trace.log 2>&1; tail -10 gpurun_out/r2m_trace.log
