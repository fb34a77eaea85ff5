HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook_seg|k_compress_s0b" -s 20 -c 2 -o gpurun_out/p63_adaptive python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 adaptive 0 1 > /dev/null 2>&1
echo done
