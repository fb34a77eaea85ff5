timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_distributed.py -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/ncu_target_multi.py rmatx:scale=28,ef=16,seed=1 8 3
python tools/ncu_target_multi.py rmatx:scale=28,ef=16,seed=1 2 3
timeout 900 python tools/scale_model.py > gpurun_out/r2_v6_scale_model.log 2>&1; echo "scale rc=$?"; cut -c1-120 gpurun_out/r2_v6_scale_model.log
