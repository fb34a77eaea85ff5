for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  for V in "" "HCC_WALK=8" "HCC_WALK=32" "HCC_WALK_LAST=2" "HCC_WALK_LAST=8" "HCC_FORMING_PCT=10" "HCC_FORMING_PCT=30" ""; do
    echo "$S [$V] $(env $V python tools/probe.py $S --reps 15 | cut -c60-120)"
  done
done
