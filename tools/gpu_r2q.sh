mkdir -p gpurun_out
for v in default prio4 norq2; do
  if [ $v = default ]; then L=""; else L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"; fi
  for c in 2 4 3; do env $L timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/r2q_var.log 2>&1; done
done
cat gpurun_out/r2q_var.log
HSIM_FULL=1 timeout 2400 python -m pytest tests/test_parity_gpu_r2.py -k exhaustive_config3 -x -q -s > gpurun_out/r2q_exh3.log 2>&1; tail -3 gpurun_out/r2q_exh3.log
