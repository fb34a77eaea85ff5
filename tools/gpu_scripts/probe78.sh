timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-120)"
done
echo "rmat28 $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 --check | cut -c60-125) $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 1 --check | grep -o 'exact[^,}]*')"
echo "shard8 $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,536870912 --reps 3 | cut -c60-125)"
