timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  for V in 1 0; do
    echo "$S settled=$V $(HCC_SETTLED=$V python tools/probe.py $S --reps 20 | cut -c60-110)"
    echo "$S adaptive settled=$V $(HCC_SETTLED=$V python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
  done
done
for V in 1 0; do
  echo "rmat28 settled=$V $(HCC_SETTLED=$V timeout 600 python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 4 --check | cut -c1-200)"
done
