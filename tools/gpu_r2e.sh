set -x
mkdir -p gpurun_out
for mc in 8 16 32; do
  for c in 2 4 3; do CUDA_DEVICE_MAX_CONNECTIONS=$mc timeout 120 python tools/variant_bench.py $c 20 2>&1 | sed "s/^/mc$mc /" >> gpurun_out/r2e_var.log; done
done
cat gpurun_out/r2e_var.log
CUDA_DEVICE_MAX_CONNECTIONS=32 HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2e_trace.log 2>&1; tail -18 gpurun_out/r2e_trace.log
