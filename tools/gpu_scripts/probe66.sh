for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1; do
  for V in "" "HCC_COMP_WIDE=1" "HCC_COMP16=1" "HCC_DYN=0" "HCC_ADAPT_PICKS=0" "HCC_ADAPT_PICKS=8"; do
    echo "$S adaptive [$V] $(env $V python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-120)"
  done
done
