timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_distributed.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/scale_model.py > gpurun_out/r2_v5_scale_model.log 2>&1; echo "scale rc=$?"; cut -c1-120 gpurun_out/r2_v5_scale_model.log
python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,536870912 --reps 3 --timeline > gpurun_out/p45_shard8.log 2>&1
head -1 gpurun_out/p45_shard8.log | cut -c1-300
timeout 600 python bench.py --force-multi --workload rmat28 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p45_rmat28_n1.json 2>gpurun_out/p45_rmat28_n1.err; echo "bench rc=$?"
