ncu --set full --clock-control none --import-source on -k k_compress_s0b -s 3 -c 1 -o gpurun_out/r2_rmat28_late_compress python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 > gpurun_out/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k k_compress_s0b -s 0 -c 1 -o gpurun_out/r2_rmat28_first_compress python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 >> gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu4.log
