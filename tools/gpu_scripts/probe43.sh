timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adaptive or golden or counters" 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  for V in 0 1 2 3 5; do
    echo "$S adaptive small=$V $(HCC_ADAPT_SMALL=$V python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-110)"
  done
done
HCC_ADAPT_SMALL=1 python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5 --timeline > gpurun_out/p43_ad_s1.log 2>&1
echo "rmat28 adaptive $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --algo adaptive --reps 2 --check | cut -c60-200)"
