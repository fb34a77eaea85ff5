timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_multi.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-110)"
  echo "$S adaptive $(python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
done
