#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_variants_gpu.py -x -q -rs -k "bucket" --durations=5 > gpurun_out/buckets11.log 2>&1; tail -12 gpurun_out/buckets11.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_overlap_gpu.py -x -q > gpurun_out/parity11.log 2>&1; tail -2 gpurun_out/parity11.log
python tools/variant_bench.py 2 20; python tools/variant_bench.py 4 10
