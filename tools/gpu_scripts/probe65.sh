timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 erx:n=16777217,m=268435456,seed=1; do
  for L in "" "HCC_LIB=paper_1612_01178_b200/lib/variants/pad33.so" "" "HCC_LIB=paper_1612_01178_b200/lib/variants/pad33.so"; do
    echo "$S [$L] $(env $L python tools/probe.py $S --reps 20 | cut -c60-120)"
  done
  echo "$S adaptive $(python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-120)"
  echo "$S adaptive pad33 $(HCC_LIB=paper_1612_01178_b200/lib/variants/pad33.so python tools/probe.py $S --algo adaptive --reps 10 | cut -c60-120)"
done
python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 10 --timeline > gpurun_out/p65.log 2>&1
