S=rmatx:scale=28,ef=16,seed=1
python tools/probe.py $S --reps 5 --forest --smi
python tools/probe.py $S --reps 5 --forest --gloo
python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 20 --smi
