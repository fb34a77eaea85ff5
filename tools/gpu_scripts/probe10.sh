S=rmatx:scale=28,ef=16,seed=1
for i in 1 2 3; do python tools/probe.py $S --reps 3 --forest | cut -c1-100; done
for i in 1 2; do python tools/probe.py $S --reps 3 --devices 0 | cut -c1-100; done
for i in 1 2; do python tools/probe.py $S --reps 3 | cut -c1-100; done
