for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-110)"
  echo "$S sumd_any $(HCC_SUMD_ANY=1 python tools/probe.py $S --reps 20 | cut -c60-110)"
done
python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 10 --timeline > gpurun_out/p36_adaptive_timeline.log 2>&1
HCC_LAUNCH=eager ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p36_adaptive_launches.csv python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 adaptive 0 2 > /dev/null 2>&1
HCC_LAUNCH=eager ncu --set full --clock-control none --import-source on -k regex:"k_hook_seg|k_compress_s0b" -s 20 -c 4 -o gpurun_out/p36_adaptive_full python tools/ncu_target.py rmatx:scale=24,ef=16,seed=1 adaptive 0 1 > /dev/null 2>&1
ncu -i gpurun_out/p36_adaptive_full.ncu-rep --page raw --csv | gzip > gpurun_out/p36_adaptive_full_raw.csv.gz
echo done
