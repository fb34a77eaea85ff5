for S in grid:4096x4096 grid:2048x2048 rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1; do
  for L in "" "HCC_LIB=paper_1612_01178_b200/lib/variants/depprog.so" "" "HCC_LIB=paper_1612_01178_b200/lib/variants/depprog.so"; do
    echo "$S [$L] $(env $L python tools/probe.py $S --reps 20 --check | cut -c60-120) $(env $L python tools/probe.py $S --reps 1 --check | grep -o 'exact[^,}]*')"
  done
  echo "$S adaptive $(python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-120)"
  echo "$S adaptive depprog $(HCC_LIB=paper_1612_01178_b200/lib/variants/depprog.so python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-120)"
done
