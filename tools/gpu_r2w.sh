mkdir -p gpurun_out
for rep in 1 2; do for v in default fm3; do
  if [ $v = default ]; then L=""; else L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"; fi
  for c in 2 4 3; do env $L timeout 120 python tools/variant_bench.py $c 30 >> gpurun_out/r2w_var.log 2>&1; done
done; done
cat gpurun_out/r2w_var.log
