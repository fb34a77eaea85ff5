S=rmatx:scale=28,ef=16,seed=1
for PAD in 0 0x100000 0x400000 0x1000000 0x2000000 0x4000000 0x8000000 0x800; do
  echo "pad $PAD $(HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
done
