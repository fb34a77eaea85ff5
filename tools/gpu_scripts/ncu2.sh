ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_ncu_rmat28_launches.csv python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k k_hook -s 2 -c 1 -o gpurun_out/r2_rmat28_steady_hook python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
