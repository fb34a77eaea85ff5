timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=16,ef=16,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-120)"
done
S=rmatx:scale=28,ef=16,seed=1
for PAD in 0 0x100000; do
echo "28 pad $PAD sumd $(HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-120)"
echo "28 pad $PAD plain $(HCC_SUMD=0 HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-120)"
done
