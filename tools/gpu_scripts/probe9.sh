S=rmatx:scale=28,ef=16,seed=1
P="python tools/probe.py"
$P $S --reps 3 --forest | cut -c1-120
$P $S --reps 3 --forest --noflush | cut -c1-120
$P $S --reps 3 --devices 0 | cut -c1-300
HCC_MULTI_SERIAL=1 $P $S --reps 3 --devices 0 | cut -c1-300
$P $S --reps 3 --forest | cut -c1-120
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory --format=csv
