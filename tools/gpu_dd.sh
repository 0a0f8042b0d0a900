set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dedup_gpu.py -x -q > gpurun_out/dd_test.log 2>&1; tail -5 gpurun_out/dd_test.log
timeout 600 python tools/dedup_timing.py 2 4 3 5 > gpurun_out/dd_timing.log 2>&1; cat gpurun_out/dd_timing.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/dd_trace.log 2>&1; tail -20 gpurun_out/dd_trace.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_dd.log 2>&1; tail -5 gpurun_out/gputest_dd.log
