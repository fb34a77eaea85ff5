for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=22,ef=16,seed=1; do
for CFG in "X=0" "HCC_FORMING_PCT=25" "HCC_FORMING_PCT=30" "HCC_FORMING_PCT=15" "HCC_PLAN=adapt:7:3" "HCC_PLAN=adapt:6:4" "HCC_PLAN=adapt:8:4" "HCC_PLAN=adapt:8:5"; do
  echo "$S $CFG $(env $CFG python tools/probe.py $S --reps 10 | cut -c60-110)"
done
done
