HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k k_hook_sumd -s 1 -c 1 -o gpurun_out/r2_sumd python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 1 > gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu5.log
