S=rmatx:scale=28,ef=16,seed=1
for PAD in 0 0x100000 0x2000000; do
  echo "pad $PAD graph  $(HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
  echo "pad $PAD eager  $(HCC_LAUNCH=eager HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
  echo "pad $PAD eagAPW $(HCC_APW=1 HCC_LAUNCH=eager HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
  echo "pad $PAD grAPW  $(HCC_APW=1 HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 | cut -c60-110)"
done
