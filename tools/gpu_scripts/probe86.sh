for S in grid:4096x4096 grid:2048x2048 erx:n=4194304,m=16777216,seed=1 rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=4,seed=1; do
  for V in "" "HCC_BOTH_LAST=1" "" "HCC_BOTH_LAST=1"; do
    echo "$S [$V] $(env $V python tools/probe.py $S --reps 20 | cut -c60-120)"
  done
  HCC_BOTH_LAST=1 python tools/probe.py $S --reps 2 --check | grep -o 'exact[^,}]*'
done
