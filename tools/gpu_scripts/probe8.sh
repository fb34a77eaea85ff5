timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
P="python tools/probe.py"
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=16,ef=16,seed=1; do
$P $S --reps 10 --check
$P $S --algo adaptive --reps 10
done
$P rmatx:scale=28,ef=16,seed=1 --reps 3 --check
$P rmatx:scale=28,ef=16,seed=1 --algo adaptive --reps 3
