for V in 1 0; do
HCC_S0B=$V python tools/probe.py grid:4096x4096 --reps 10 --timeline > gpurun_out/p52_$V.log 2>&1
HCC_S0B=$V python tools/probe.py rmatx:scale=16,ef=16,seed=1 --reps 10 --timeline > gpurun_out/p52_r16_$V.log 2>&1
done
