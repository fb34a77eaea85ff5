for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096 rmatx:scale=22,ef=16,seed=1 erx:n=4194304,m=16777216,seed=1; do
  for L in "" "HCC_LIB=paper_1612_01178_b200/lib/variants/both768e4.so" "" "HCC_LIB=paper_1612_01178_b200/lib/variants/both768e4.so"; do
    echo "$S [$L] $(env $L python tools/probe.py $S --reps 30 | cut -c60-120)"
  done
done
