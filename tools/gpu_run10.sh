#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_variants_gpu.py -x -q -rs --durations=8 > gpurun_out/variants10.log 2>&1; tail -15 gpurun_out/variants10.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_overlap_gpu.py -x -q > gpurun_out/parity10.log 2>&1; tail -3 gpurun_out/parity10.log
python tools/variant_bench.py 2 20; python tools/variant_bench.py 4 10
