mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_split" -s 1 -c 1 -o gpurun_out/prof_split_v9 python tools/prof_sweep.py 2 2 > gpurun_out/r2r_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pipe<4>|k_pipe_cont" -s 2 -c 2 -o gpurun_out/prof_pipe4_v9 python tools/prof_sweep.py 2 2 >> gpurun_out/r2r_ncu.log 2>&1
tail -2 gpurun_out/r2r_ncu.log
