timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 erx:n=67108864,m=1073741824,seed=3 grid:4096x4096; do
  echo "$S $(python tools/probe.py $S --reps 10 | cut -c60-110)"
done
echo "adaptive $(python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 10 | cut -c60-110)"
