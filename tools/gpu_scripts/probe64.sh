for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096 erx:n=4194304,m=16777216,seed=1; do
  for V in "" "HCC_ADAPT_GROWTH=2 HCC_PLAN=adapt:7:6" "HCC_ADAPT_GROWTH=2 HCC_PLAN=adapt:7:8" "HCC_ADAPT_GROWTH=3 HCC_PLAN=adapt:7:5" "HCC_PLAN=adapt:7:6" "HCC_PLAN=adapt:8:6" "HCC_ADAPT_GROWTH=2 HCC_PLAN=adapt:8:8"; do
    echo "$S [$V] $(env $V python tools/probe.py $S --reps 15 | cut -c60-125)"
  done
done
