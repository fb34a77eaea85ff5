P="python tools/probe.py"
for V in "" bl2 pig bl2pig; do
  if [ -n "$V" ]; then export HCC_LIB=paper_1612_01178_b200/lib/variants/$V.so; else unset HCC_LIB; fi
  echo "== variant ${V:-default}"
  $P rmatx:scale=28,ef=16,seed=1 --reps 3 | cut -c1-200
  $P rmatx:scale=24,ef=16,seed=1 --reps 10 | cut -c1-200
  $P erx:n=16777216,m=268435456,seed=1 --reps 5 | cut -c1-200
done
