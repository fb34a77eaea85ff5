for S in rmatx:scale=16,ef=16,seed=1 rmatx:scale=17,ef=16,seed=1 rmatx:scale=18,ef=16,seed=1 rmatx:scale=20,ef=16,seed=1 erx:n=262144,m=4194304,seed=1 grid:512x512 grid:1024x1024; do
  for V in 1 0; do
    echo "$S s0b=$V $(HCC_S0B=$V python tools/probe.py $S --reps 30 | cut -c60-125)"
  done
  echo "$S s0b=1 plan7:3 $(HCC_PLAN=adapt:7:3 python tools/probe.py $S --reps 30 | cut -c60-125)"
  echo "$S s0b=0 plan7:3 $(HCC_S0B=0 HCC_PLAN=adapt:7:3 python tools/probe.py $S --reps 30 | cut -c60-125)"
done
