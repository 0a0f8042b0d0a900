mkdir -p gpurun_out
for v in mm0 mlp mg2 mg4; do
  L="HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so"
  for c in 2 4 3; do env $L timeout 120 python tools/variant_bench.py $c 20 >> gpurun_out/r2i_var.log 2>&1; done
done
cat gpurun_out/r2i_var.log
