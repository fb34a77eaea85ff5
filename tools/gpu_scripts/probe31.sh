for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 erx:n=16777217,m=268435456,seed=2 grid:4096x4096; do
 for W in 1 0; do
  echo "$S wl_sumd=$W $(HCC_WL_SUMD=$W python tools/probe.py $S --reps 10 --timeline --check | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact'), end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
")"
 done
done
