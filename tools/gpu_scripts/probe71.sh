HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook|k_compress_s0b" -c 8 -o gpurun_out/p71_er python tools/ncu_target.py erx:n=16777216,m=268435456,seed=1 baseline-mj 0 1 > /dev/null 2>&1
echo done
