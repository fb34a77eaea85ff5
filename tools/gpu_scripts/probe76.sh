for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 rmatx:scale=20,ef=16,seed=7; do
  for V in "" "HCC_ADAPT_HALF=1" "" "HCC_ADAPT_HALF=1"; do
    echo "$S adaptive [$V] $(env $V python tools/probe.py $S --algo adaptive --reps 10 --check | cut -c60-125) $(env $V python tools/probe.py $S --algo adaptive --reps 2 --check | grep -o 'exact[^,}]*')"
  done
done
