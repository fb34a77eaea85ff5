for V in "" sh0 swz1 sh0swz1 ""; do
  if [ -n "$V" ]; then export HCC_LIB=paper_1612_01178_b200/lib/variants/$V.so; else unset HCC_LIB; fi
  echo "${V:-default} $(python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 20 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d['ms_min'], end=' :: '); continue
    print(round(d['hook_ms'],4), end=' | ')
") ER $(python tools/probe.py erx:n=16777216,m=268435456,seed=1 --reps 10 | cut -c72-90)"
done
