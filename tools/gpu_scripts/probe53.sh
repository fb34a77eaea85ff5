S=rmatx:scale=28,ef=16,seed=1
for V in 1 0; do
  echo "shard8 s0b=$V $(HCC_S0B=$V python tools/probe.py $S --range 0,536870912 --reps 3 | cut -c60-125)"
  echo "shard4 s0b=$V $(HCC_S0B=$V python tools/probe.py $S --range 0,1073741824 --reps 3 | cut -c60-125)"
done
for S in erx:n=4194304,m=16777216,seed=1 erx:n=16777216,m=67108864,seed=2 rmatx:scale=24,ef=4,seed=1 rmatx:scale=22,ef=8,seed=1 erx:n=16777216,m=134217728,seed=2 grid:8192x4096; do
  for V in 1 0; do
    echo "$S s0b=$V $(HCC_S0B=$V python tools/probe.py $S --reps 10 | cut -c60-125)"
  done
done
