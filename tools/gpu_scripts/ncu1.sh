ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_ncu_adaptive_rmat24_launches.csv python tools/ncu_run.py rmatx:scale=24,ef=16,seed=1 adaptive 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hook_seg_cas -s 0 -c 2 -o gpurun_out/r2_adaptive_seg_cas python tools/ncu_run.py rmatx:scale=24,ef=16,seed=1 adaptive 1 > gpurun_out/ncu1.log 2>&1
ls -la gpurun_out/
