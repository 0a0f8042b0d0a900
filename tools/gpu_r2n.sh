mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dedup_gpu.py tests/test_parity_gpu.py tests/test_parity_gpu_r2.py -x -q > gpurun_out/r2n_test.log 2>&1; tail -2 gpurun_out/r2n_test.log
for v in on off; do
  if [ $v = off ]; then E="HSIM_SEED_OFF=1"; else E="X=1"; fi
  for c in 2 4 3; do env $E timeout 120 python tools/variant_bench.py $c 20 2>&1 | sed "s/^/seed-$v /" >> gpurun_out/r2n_var.log; done
done
cat gpurun_out/r2n_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2n_trace.log 2>&1; tail -10 gpurun_out/r2n_trace.log
