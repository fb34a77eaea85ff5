for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096; do
  python tools/probe.py $S --reps 10 --timeline > gpurun_out/p47_$(echo $S | cut -c1-4).log 2>&1
done
