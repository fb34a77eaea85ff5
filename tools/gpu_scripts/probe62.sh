ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p62_multi8.csv python tools/ncu_target_multi.py rmatx:scale=28,ef=16,seed=1 8 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_merge_gather -c 1 -o gpurun_out/p62_gather python tools/ncu_target_multi.py rmatx:scale=28,ef=16,seed=1 8 1 > /dev/null 2>&1
echo done
