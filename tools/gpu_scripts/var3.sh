for V in "" swz2 "" swz2; do
  if [ -n "$V" ]; then export HCC_LIB=paper_1612_01178_b200/lib/variants/$V.so; else unset HCC_LIB; fi
  echo "${V:-default} $(python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 20 --check | cut -c60-110) ER $(python tools/probe.py erx:n=16777216,m=268435456,seed=1 --reps 10 --check | cut -c72-90)"
done
