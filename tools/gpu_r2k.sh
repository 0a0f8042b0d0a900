mkdir -p gpurun_out
for c in 2 4 3; do timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/r2k_var.log 2>&1; done
cat gpurun_out/r2k_var.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_test.log 2>&1; tail -3 gpurun_out/r2k_test.log
timeout 600 python tools/dedup_timing.py 5 > gpurun_out/r2k_c5.log 2>&1; cat gpurun_out/r2k_c5.log
