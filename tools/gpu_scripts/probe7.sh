P="python tools/probe.py"
$P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 10 --check
HCC_SEG_CAS=0 $P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 10
$P erx:n=16777216,m=268435456,seed=1 --algo adaptive --reps 5 --check
$P grid:4096x4096 --algo adaptive --reps 5 --check
$P rmatx:scale=28,ef=16,seed=1 --algo adaptive --reps 3
$P rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 3 --timeline | tail -12
