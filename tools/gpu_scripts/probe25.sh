for S in rmatx:scale=26,ef=16,seed=1 rmatx:scale=28,ef=16,seed=1 rmatx:scale=24,ef=16,seed=1 erx:n=16777217,m=268435456,seed=2; do
  R=5; case $S in *28*) R=3;; esac
  echo "$S $(python tools/probe.py $S --reps $R | cut -c60-120)"
done
