#!/bin/bash
# f4 variants on the GPU: parity tests, then the full GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_variants_gpu.py -x -q -rs --durations=10 > gpurun_out/variants5.log 2>&1; tail -25 gpurun_out/variants5.log
