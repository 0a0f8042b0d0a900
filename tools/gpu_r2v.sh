mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_r2.py tests/test_dedup_gpu.py -x -q > gpurun_out/r2v_test.log 2>&1; tail -1 gpurun_out/r2v_test.log
for rep in 1 2; do for c in 2 4 3; do timeout 120 python tools/variant_bench.py $c 30 >> gpurun_out/r2v_var.log 2>&1; done; done
cat gpurun_out/r2v_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2v_trace.log 2>&1; tail -4 gpurun_out/r2v_trace.log
