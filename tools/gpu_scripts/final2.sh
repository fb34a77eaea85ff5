timeout 1200 python bench.py > gpurun_out/r2_bench_v2.json 2> gpurun_out/r2_bench_v2.err; echo "bench rc=$?"
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_v2_launches_rmat24_eager.csv python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 2 > /dev/null 2>&1
HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook|k_compress|k_start|k_step|k_star" -c 24 -o gpurun_out/r2_v2_rmat24_full python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 1 > gpurun_out/r2_v2_ncu_full.log 2>&1
ncu -i gpurun_out/r2_v2_rmat24_full.ncu-rep --page raw --csv | gzip > gpurun_out/r2_v2_rmat24_full_raw.csv.gz
timeout 900 python tools/scale_model.py > gpurun_out/r2_v2_scale_model.log 2>&1
cp profiles/r2_rmat28_scaling_model.json gpurun_out/r2_v2_rmat28_scaling_model.json
tail -c 600 gpurun_out/r2_bench_v2.json
