timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 erx:n=16777217,m=268435456,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-110)"
  echo "$S adaptive $(python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
done
python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5 --timeline > gpurun_out/p44_ad.log 2>&1
