for V in 0 1; do
  HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 --timeline > gpurun_out/p79_$V.log 2>&1
  HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,536870912 --reps 3 --timeline > gpurun_out/p79s_$V.log 2>&1
  HCC_HOOK_BOTH=$V python tools/probe.py rmatx:scale=28,ef=16,seed=1 --range 0,2147483648 --reps 3 --timeline > gpurun_out/p79h_$V.log 2>&1
done
