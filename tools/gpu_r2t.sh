mkdir -p gpurun_out
for rep in 1 2; do
for v in default mfirst prio4; do
  if [ $v = default ]; then L=""; else L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"; fi
  for c in 2 4 3; do env $L timeout 120 python tools/variant_bench.py $c 30 >> gpurun_out/r2t_var.log 2>&1; done
done
done
cat gpurun_out/r2t_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2t_trace.log 2>&1; tail -10 gpurun_out/r2t_trace.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dedup_gpu.py -x -q > gpurun_out/r2t_test.log 2>&1; tail -1 gpurun_out/r2t_test.log
