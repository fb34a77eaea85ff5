timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in grid:4096x4096 rmatx:scale=16,ef=16,seed=1 rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 erx:n=4194304,m=16777216,seed=1 rmatx:scale=20,ef=16,seed=1 grid:1024x1024 erx:n=1048576,m=16777216,seed=1; do
  for V in "HCC_BITS_GATE=0" "HCC_BITS_GATE=1" "HCC_BUILD_PCT=15" "HCC_BUILD_PCT=40"; do
    echo "$S [$V] $(env $V python tools/probe.py $S --reps 20 | cut -c60-120)"
  done
done
echo "shard8 $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,536870912 --reps 3 | cut -c60-125)"
echo "rmat28 $(python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 | cut -c60-125)"
