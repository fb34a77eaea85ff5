timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-120)"
done
