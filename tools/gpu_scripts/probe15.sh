timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
S=rmatx:scale=28,ef=16,seed=1
for PAD in 0 0x100000 0x2000000; do
  echo "pad $PAD dyn  $(HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
  echo "pad $PAD stat $(HCC_DYN=0 HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
done
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  echo "$S dyn  $(python tools/probe.py $S --reps 10 | cut -c40-110)"
  echo "$S stat $(HCC_DYN=0 python tools/probe.py $S --reps 10 | cut -c40-110)"
  echo "$S adaptive dyn  $(python tools/probe.py $S --reps 10 --algo adaptive | cut -c40-110)"
done
