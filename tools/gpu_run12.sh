#!/bin/bash
# exhaustive config-3 parity (62.2 M candidates, compact oracle on the host cores)
mkdir -p gpurun_out
nproc
HSIM_FULL=1 timeout 3000 python -m pytest tests/test_parity_gpu_r2.py -q -s -k exhaustive_config3 > gpurun_out/full3.log 2>&1; tail -5 gpurun_out/full3.log
