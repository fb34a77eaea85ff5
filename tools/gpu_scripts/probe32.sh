timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=28,ef=16,seed=1; do
 for F in 1 0; do
  R=10; case $S in *28*) R=3;; esac
  echo "$S fold=$F $(HCC_FOLD_PICK=$F python tools/probe.py $S --reps $R | cut -c60-120)"
 done
done
