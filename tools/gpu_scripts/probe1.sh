set -x
P="python tools/probe.py"
$P rmatx:scale=28,ef=16,seed=1 --reps 3 --timeline
$P rmatx:scale=28,ef=16,seed=1 --reps 3 --forest
HCC_WL_DIV=1 $P rmatx:scale=28,ef=16,seed=1 --reps 3
HCC_HOOK_CAS=0 $P rmatx:scale=28,ef=16,seed=1 --reps 3
$P rmatx:scale=24,ef=16,seed=1 --reps 10 --timeline
$P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 5 --check --timeline
HCC_CAS_STREAM=0 $P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 3
$P erx:n=16777216,m=268435456,seed=1 --algo adaptive --reps 5 --check
$P erx:n=16777216,m=268435456,seed=1 --reps 5
$P grid:4096x4096 --algo adaptive --reps 5 --check
$P grid:4096x4096 --reps 5
