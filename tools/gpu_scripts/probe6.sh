timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -4
P="python tools/probe.py"
$P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5 --check --timeline | head -8
HCC_ADAPT_PICKS=0 $P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5
$P erx:n=16777216,m=268435456,seed=1 --algo adaptive --reps 5
$P grid:4096x4096 --algo adaptive --reps 5
$P rmatx:scale=16,ef=16,seed=1 --algo adaptive --reps 20
$P rmatx:scale=16,ef=16,seed=1 --reps 20
$P rmatx:scale=28,ef=16,seed=1 --algo adaptive --reps 3
