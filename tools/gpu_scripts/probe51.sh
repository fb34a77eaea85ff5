for S in rmatx:scale=19,ef=16,seed=1 erx:n=1048576,m=16777216,seed=1 grid:2048x2048 grid:4096x4096 erx:n=16777216,m=268435456,seed=1 rmatx:scale=22,ef=16,seed=1 erx:n=524288,m=2097152,seed=3; do
  for V in 1 0; do
    echo "$S s0b=$V $(HCC_S0B=$V python tools/probe.py $S --reps 20 | cut -c60-125)"
  done
done
