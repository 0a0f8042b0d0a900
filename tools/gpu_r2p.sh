mkdir -p gpurun_out
for v in default prio4 fm2; do
  if [ $v = default ]; then L=""; else L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"; fi
  for c in 2 4 3; do env $L timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/r2p_var.log 2>&1; done
done
cat gpurun_out/r2p_var.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_test.log 2>&1; tail -2 gpurun_out/r2p_test.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2p_trace.log 2>&1; tail -10 gpurun_out/r2p_trace.log
