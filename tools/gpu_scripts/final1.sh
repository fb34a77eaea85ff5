# round-2 measurement session: tests, smoke, bench, launch lists, ncu, scaling model
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest_final.log
tail -3 gpurun_out/r2_gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; tail -1 gpurun_out/r2_smoke_final.log
timeout 1200 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; echo "ref rc=$?"
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat24_eager.csv python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 2 > /dev/null 2>&1
HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook|k_compress|k_start|k_step|k_star" -c 24 -o gpurun_out/r2_rmat24_full python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 1 > gpurun_out/r2_ncu_full.log 2>&1
ncu -i gpurun_out/r2_rmat24_full.ncu-rep --page raw --csv | gzip > gpurun_out/r2_rmat24_full_raw.csv.gz
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat28_eager.csv python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_adaptive_rmat24_eager.csv python tools/ncu_run.py rmatx:scale=24,ef=16,seed=1 adaptive 1 > /dev/null 2>&1
timeout 900 python tools/scale_model.py > gpurun_out/r2_scale_model.log 2>&1
cp profiles/r2_rmat28_scaling_model.json gpurun_out/ 2>/dev/null
ls -la gpurun_out
