S=rmatx:scale=24,ef=16,seed=1
for V in "" sumd768 sumd512; do
  if [ -n "$V" ]; then export HCC_LIB=paper_1612_01178_b200/lib/variants/$V.so; else unset HCC_LIB; fi
  echo "${V:-sumd1024} $(HCC_SUMD=1 python tools/probe.py $S --reps 10 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], end=' :: '); continue
    print(round(d['hook_ms'],4), end=' | ')
")"
done
unset HCC_LIB
echo "plain $(python tools/probe.py $S --reps 10 | cut -c60-110)"
