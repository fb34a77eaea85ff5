timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 erx:n=16777217,m=268435456,seed=2 grid:4096x4096 rmatx:scale=16,ef=16,seed=1 rmatx:scale=20,ef=16,seed=1 rmatx:scale=28,ef=16,seed=1; do
  R=10; case $S in *28*) R=3;; esac
  echo "$S $(python tools/probe.py $S --reps $R | cut -c60-120)"
done
echo "adaptive $(python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5 | cut -c60-120)"
