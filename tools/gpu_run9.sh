#!/bin/bash
mkdir -p gpurun_out
for g in 0 1 2 3 4 6; do
  for c in 2 4; do HSIM_SYNC_FIRST=$g python tools/variant_bench.py $c 20 | sed "s/^/sf=$g /"; done
done
HSIM_SYNC_FIRST=2 HSIM_TRACE=1 python tools/trace_sweep.py 2 3 2> gpurun_out/trace9.log; grep -A40 "call 2" gpurun_out/trace9.log
HSIM_SYNC_FIRST=2 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
