timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 4 --timeline --check > gpurun_out/p41_r28.log 2>&1
head -1 gpurun_out/p41_r28.log | cut -c1-330
grep -i check gpurun_out/p41_r28.log | head -3
python tools/probe.py rmatx:scale=28,ef=16,seed=1 --algo adaptive --reps 2 | cut -c1-200
python tools/probe.py erx:n=67108864,m=1073741824,seed=1 --reps 4 | cut -c1-200
HCC_SUM_MAX_SHIFT=6 python tools/probe.py erx:n=67108864,m=1073741824,seed=1 --reps 4 | cut -c1-200
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-110)"
  echo "$S adaptive $(python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
done
