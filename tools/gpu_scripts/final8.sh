timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest9.log
tail -2 gpurun_out/r2_gputest9.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r2_bench_v7.json 2> gpurun_out/r2_bench_v7.err; echo "bench rc=$?"
for W in er24 grid4096 rmat16; do timeout 900 python bench.py --workload $W --no-rmat28 --no-adaptive --e2e-steps 2 > gpurun_out/r2_bench_v7_$W.json 2>/dev/null; echo "$W rc=$?"; done
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_v7_launches_rmat24_eager.csv python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 2 > /dev/null 2>&1
HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook|k_compress|k_start|k_step|k_star" -c 26 -o gpurun_out/r2_v7_rmat24_full python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 baseline-mj 0 1 > /dev/null 2>&1
ncu -i gpurun_out/r2_v7_rmat24_full.ncu-rep --page raw --csv | gzip > gpurun_out/r2_v7_rmat24_full_raw.csv.gz
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_v7_launches_adaptive_eager.csv python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 adaptive 0 2 > /dev/null 2>&1
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_v7_launches_rmat28_eager.csv python tools/ncu_target.py rmatx:scale=28,ef=16,seed=1 baseline-mj 0 1 > /dev/null 2>&1
echo done
