for V in 0 1; do
  echo "rmat28 both=$V $(HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 | cut -c60-125)"
  echo "shard8 both=$V $(HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,536870912 --reps 3 | cut -c60-125)"
  echo "shard2 both=$V $(HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,2147483648 --reps 3 | cut -c60-125)"
  echo "er26 both=$V $(HCC_HOOK_BOTH=$V python tools/probe.py erx:n=67108864,m=1073741824,seed=1 --reps 3 | cut -c60-125)"
done
