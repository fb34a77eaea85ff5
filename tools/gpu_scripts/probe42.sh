HCC_COMP16=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  for V in 1 0 1 0; do
    echo "$S c16=$V $(HCC_COMP16=$V python tools/probe.py $S --reps 20 | cut -c60-110)"
    echo "$S adaptive c16=$V $(HCC_COMP16=$V python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
  done
done
for V in 1 0; do
  echo "rmat28 c16=$V $(HCC_COMP16=$V timeout 600 python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 4 --check | cut -c60-330)"
done
