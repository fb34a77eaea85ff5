S=rmatx:scale=28,ef=16,seed=1
for V in "" "HCC_PLAN=adapt:6" "HCC_PLAN=adapt:5" "HCC_PLAN=adapt:4" "HCC_PLAN=adapt:5:3" "HCC_PLAN=adapt:8" "HCC_PLAN_NSHIFT=4" "HCC_PLAN_NSHIFT=3" "HCC_FORMING_PCT=10" "HCC_FORMING_PCT=35"; do
  echo "shard8 [$V] $(env $V python tools/probe.py $S --range 0,536870912 --reps 3 | cut -c60-200)"
done
for V in "" "HCC_PLAN=adapt:5" "HCC_PLAN_NSHIFT=4"; do
  echo "shard2 [$V] $(env $V python tools/probe.py $S --range 0,2147483648 --reps 3 | cut -c60-200)"
done
