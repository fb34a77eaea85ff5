timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adaptive or golden or engine or wide or steady" 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=20,ef=16,seed=1; do
  echo "$S sumd $(python tools/probe.py $S --algo adaptive --reps 10 --check | cut -c60-140)"
  echo "$S plain $(HCC_SEG_SUMD=0 python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-140)"
done
