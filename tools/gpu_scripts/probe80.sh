timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096 rmatx:scale=22,ef=16,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-120)"
  echo "$S off $(HCC_HOOK_BOTH=0 python tools/probe.py $S --reps 20 | cut -c60-120)"
done
echo "rmat28 $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 | cut -c60-125)"
