mkdir -p gpurun_out
for v in mm0 mp8 mp9; do
  L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"
  for c in 3 2; do env $L timeout 120 python tools/variant_bench.py $c 10 >> gpurun_out/r2j_var.log 2>&1; done
done
cat gpurun_out/r2j_var.log
