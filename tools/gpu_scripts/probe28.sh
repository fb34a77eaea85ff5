for V in "" sumstatic; do
  if [ -n "$V" ]; then export HCC_LIB=paper_1612_01178_b200/lib/variants/$V.so; else unset HCC_LIB; fi
  for S in erx:n=16777217,m=268435456,seed=2 erx:n=67108864,m=268435456,seed=3 erx:n=67108864,m=1073741824,seed=3; do
    echo "${V:-dyn} $S $(python tools/probe.py $S --reps 5 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
")"
  done
done
