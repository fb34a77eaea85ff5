for PF in 0 888 1776 444 3552; do
  HCC_COMP_PF=$PF python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 --timeline > gpurun_out/p39_r28_pf$PF.log 2>&1
  echo "rmat28 pf=$PF $(head -1 gpurun_out/p39_r28_pf$PF.log | cut -c60-200)"
done
for PF in 0 888; do
  echo "rmat24 pf=$PF $(HCC_COMP_PF=$PF python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 20 | cut -c60-110)"
done
