HCC_LAUNCH=eager ncu --set full --clock-control none -k regex:"^k_hook$" -s 2 -c 1 -o gpurun_out/r2_v6_rmat28_steady python tools/ncu_target.py rmatx:scale=28,ef=16,seed=1 baseline-mj 0 1 > gpurun_out/p73.log 2>&1
echo rc=$?
