mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dedup_gpu.py tests/test_parity_gpu.py tests/test_parity_gpu_r2.py -x -q > gpurun_out/r2s_test.log 2>&1; tail -2 gpurun_out/r2s_test.log
for c in 2 4 3; do timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/r2s_var.log 2>&1; done
cat gpurun_out/r2s_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2s_trace.log 2>&1; tail -4 gpurun_out/r2s_trace.log
