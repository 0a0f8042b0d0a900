#!/bin/bash
# Times the default library and the listed variants on configs (args: variant names).
for c in ${CONFIGS:-2 3 4}; do
  python tools/variant_bench.py $c 10
  for v in "$@"; do HSIM_LIB=paper_2508_05370_b200/variants/libhsim_$v.so python tools/variant_bench.py $c 10; done
done
