S=rmatx:scale=16,ef=16,seed=1
for V in "" "HCC_PLAN=adapt:7:1" "HCC_PLAN=adapt:7:2" "HCC_PLAN=adapt:4:2" "HCC_PLAN=adapt:2:2" "HCC_PLAN=adapt:7:3" "HCC_S0B=0"; do
  python tools/probe.py $S --reps 30 --timeline > gpurun_out/p49.log 2>&1
  echo "[$V] $(env $V python tools/probe.py $S --reps 30 | cut -c60-130)"
done
python tools/probe.py $S --reps 30 --timeline > gpurun_out/p49.log 2>&1
