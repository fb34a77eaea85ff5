HCC_S0F=0 python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 --timeline > gpurun_out/p40_r28_nos0f.log 2>&1
head -1 gpurun_out/p40_r28_nos0f.log | cut -c60-200
HCC_LAUNCH=eager ncu --set full --clock-control none -k regex:"k_compress_s0b" -s 2 -c 1 -o gpurun_out/p40_r28_comp python tools/ncu_target.py rmatx:scale=28,ef=16,seed=1 baseline-mj 0 1 > /dev/null 2>&1
ncu -i gpurun_out/p40_r28_comp.ncu-rep --page raw --csv | gzip > gpurun_out/p40_r28_comp_raw.csv.gz
echo done
