S=rmatx:scale=28,ef=16,seed=1
python tools/probe.py $S --reps 3 | cut -c1-100
python tools/probe.py $S --reps 3 --thread | cut -c1-100
python tools/probe.py $S --reps 3 --extractx | cut -c1-100
python tools/probe.py $S --reps 3 --devices 0 | cut -c1-100
